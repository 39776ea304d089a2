// Internal structures of the B200 plan-exploration engine (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>
#include <vector>

#include "../../include/autoplan_b200.h"

// Control block of the graph-capturable vectorised driver: int64[AP_CTL_WORDS]
// read by the *_ctl entry points instead of by-value step counters.
enum { AP_CTL_STEP = 0, AP_CTL_SLOT = 1, AP_CTL_SIZE = 2, AP_CTL_TRAIN = 3, AP_CTL_WORDS = 4 };

namespace apb {

void set_error(const std::string& msg);
int cuda_fail(cudaError_t err, const char* what);

#define AP_CUDA_CHECK(expr)                                   \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::apb::cuda_fail(_e, #expr); \
  } while (0)

// Programmatic dependent launch (PDL) for the chains of small dependent
// kernels (the DQN vector step): a kernel launched through launch_pdl may be
// scheduled while its predecessor in the stream is still finishing; every
// such kernel starts with pdl_entry(), which releases its own dependents and
// then waits until the predecessor has completed and its writes are visible
// (griddepcontrol is a no-op for a normally launched kernel).  AP_NO_PDL=1
// launches normally.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_entry() {
  pdl_trigger();
  pdl_wait();
}

bool pdl_enabled();
#endif

// SM count of the current device, cached per device ordinal (thread-safe: a
// racing first call stores the same value).
int current_sm_count(int* sms);

// Per-device grow-only configuration value (kernel attributes such as the
// dynamic shared-memory limit are per device context): `need(dev, v)` is true
// when v exceeds what was configured on `dev`, and records v.
struct PerDeviceMax {
  std::atomic<int64_t> v[64];
  bool need(int dev, int64_t want) {
    std::atomic<int64_t>& slot = v[dev & 63];
    int64_t cur = slot.load(std::memory_order_relaxed);
    while (want > cur)
      if (slot.compare_exchange_weak(cur, want)) return true;
    return false;
  }
};
inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}

#ifdef __CUDACC__

// Throughput-mode Adam element (the graph-captured learner; the parity agent's
// ap_dqn_adam keeps the reference expression), shared by the Adam kernels and
// the GEMM epilogue that fuses the first layer's update: explicitly rounded
// operations (never contracted, so every kernel computes the same bits),
// reciprocal bias corrections ic1 = 1/(1 - b1^t), ic2 = 1/(1 - b2^t), one fast divide.
__device__ __forceinline__ void adam_math(float gi, float& mi, float& vi, float& pi, float lr, float b1, float b2,
                                          float eps, float ic1, float ic2) {
  mi = __fadd_rn(__fmul_rn(b1, mi), __fmul_rn(1.0f - b1, gi));
  vi = __fadd_rn(__fmul_rn(b2, vi), __fmul_rn(__fmul_rn(1.0f - b2, gi), gi));
  const float den = __fadd_rn(__fsqrt_rn(__fmul_rn(vi, ic2)), eps);
  pi = __fsub_rn(pi, __fdividef(__fmul_rn(lr, __fmul_rn(mi, ic1)), den));
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
#endif

// Device buffer owned by a handle.
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  int upload(const std::vector<T>& host) {
    n = host.size();
    if (n == 0) return AP_OK;
    AP_CUDA_CHECK(cudaMalloc(&ptr, n * sizeof(T)));
    AP_CUDA_CHECK(cudaMemcpy(ptr, host.data(), n * sizeof(T), cudaMemcpyHostToDevice));
    return AP_OK;
  }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
  }
};

// One compiled rule of the reference sweep (sharding.py:155-202), kept only for
// the exact-order trace kernel.  Program words: kind, site, then operands.
enum RuleKind : int32_t { RULE_LINK = 0, RULE_DOT = 1, RULE_REDUCE = 2 };

struct GraphTables {
  // host copies
  int32_t num_instr = 0;
  int64_t num_slots = 0;
  int32_t num_classes = 0;
  int32_t num_links = 0;
  std::vector<int64_t> slot_base;     // [N+1]
  std::vector<int32_t> slot_owner;    // [S] position owning the slot
  std::vector<int32_t> class_of_slot; // [S]
  std::vector<uint8_t> slot_forced;   // [S] directly forced replicated
  std::vector<uint8_t> class_forced;  // [C]
  std::vector<int32_t> imp_offset;    // [C+1]
  std::vector<int32_t> imp_target;    // [T]
  std::vector<uint32_t> forced_words; // [ceil(C/32)] forced-replicated class bitset (generic kernel)
  std::vector<int32_t> program;       // trace program (reference sweep order)
  std::vector<int32_t> forced_list;   // forced slots in reference order

  // fast-kernel tables (only when num_classes <= kMaxFastClasses)
  bool fast = false;
  std::vector<uint32_t> slot_desc;    // [nq_s * 4] chunk descriptors (see propagate_fast.cu)
  std::vector<uint32_t> slot_desc_t;  // [nq_s * 4] same classes, transposed selectors (packed 2-bit output)
  std::vector<uint8_t> slot_cls8;     // [nq_s * 16] class id per slot, 0xFF padding
  std::vector<uint32_t> imp_bits;     // [C * 8] 256-bit implication row per class
  std::vector<uint32_t> forced_bits;  // [8] forced-replicated classes
  bool slot_all_k4 = false;           // every slot chunk has <= 4 classes, none falls back
  int32_t slot_fallback_chunks = 0;

  // device copies
  DevBuf<uint32_t> d_slot_desc;
  DevBuf<uint32_t> d_slot_desc_t;
  DevBuf<uint8_t> d_slot_cls8;
  DevBuf<uint32_t> d_imp_bits;
  DevBuf<uint32_t> d_forced_bits;
  DevBuf<int32_t> d_slot_class;
  DevBuf<uint32_t> d_forced_words;
  DevBuf<int32_t> d_imp_offset;
  DevBuf<int32_t> d_imp_target;
  // generic kernel: global per-warp P/R bitset scratch when shared memory is too small (grow-only)
  mutable uint32_t* d_scratch = nullptr;
  mutable int64_t scratch_words = 0;
  DevBuf<int32_t> d_program;
  DevBuf<int32_t> d_forced_list;
  DevBuf<int64_t> d_slot_base;
  DevBuf<int32_t> d_slot_owner;
  int device = 0;
  bool uploaded = false;
};

struct DecisionTables {
  int32_t n = 0;
  std::vector<int64_t> slots;
  std::vector<int32_t> dec_class;
  std::vector<uint8_t> dec_flags;     // bit0 candidate, bit1 slot directly forced
  std::vector<int32_t> first_same;    // [n] first position on the same tensor (U-seed pin rule)
  // fast-kernel tables
  bool fast = false;
  int32_t ncand = 0;
  std::vector<uint32_t> dec_desc;     // [nq_d * 8] chunk descriptors
  std::vector<uint32_t> dec_masks;    // [nq_d] valid | candidate << 16 (permuted bit order)
  std::vector<uint8_t> dec_cls8;      // [nq_d * 16]
  std::vector<uint16_t> class_ncand;  // [C] candidate positions per class
  std::vector<uint32_t> ncand_planes; // [16][4] lane kernel (<= 128 classes): classes whose ncand has bit k
  DevBuf<uint32_t> d_dec_desc;
  DevBuf<uint32_t> d_dec_masks;
  DevBuf<uint8_t> d_dec_cls8;
  DevBuf<uint16_t> d_class_ncand;
  DevBuf<uint32_t> d_ncand_planes;
  DevBuf<int32_t> d_dec_class;
  DevBuf<uint8_t> d_dec_flags;
  DevBuf<int32_t> d_first_same;
  DevBuf<int64_t> d_slots;
  const GraphTables* graph = nullptr;
  bool uploaded = false;
};

int build_graph(const ap_graph_desc* desc, GraphTables* g);
int ensure_graph_on_device(GraphTables* g);
int ensure_decision_on_device(DecisionTables* d);
int build_decision(const GraphTables* g, const int64_t* slots, const uint8_t* is_cand, int32_t n,
                   DecisionTables* d);

constexpr int kMaxFastClasses = 255;  // class 255 is the padding marker of the fast tables
constexpr int kFastMaxChunks = 8;     // decision positions <= 32 lanes * 8 chunks * 16

void build_fast_graph(GraphTables* g);
void build_fast_decision(const GraphTables* g, DecisionTables* d);
// Returns AP_ERR_UNSUPPORTED (without setting an error) when the fast path does not apply.
// `packed_out` (nullable, [batch, packed_stride] bytes): slot statuses at 2 bits per slot
// (code = status + 1, slot j in bits 2*(j%16) of 32-bit word j/16), exclusive with slots_out.
int launch_propagate_fast(const GraphTables* g, const DecisionTables* d, const int8_t* seeds, int64_t batch,
                          int64_t seed_stride, int8_t* slots_out, int64_t slots_stride, int8_t* cand_out,
                          int64_t cand_stride, uint8_t* outcome, int32_t* counts, cudaStream_t stream,
                          uint8_t* packed_out = nullptr, int64_t packed_stride = 0);

int launch_gemm_v2(const float* A, int64_t lda, int transA, const float* B, int64_t ldb, int transB, float* C,
                   int64_t ldc, int M, int N, int K, const float* bias, int relu, int precision, cudaStream_t stream);
// Split-K partials workspace of at least `bytes`, one per stream (concurrent
// GEMMs on parallel graph branches never share it).  Grow-only: a captured
// graph may hold an older buffer, so none is freed, and none grows inside a
// capture (AP_ERR_INVALID then; warm the shapes up eagerly first).
int splitk_workspace(cudaStream_t stream, size_t bytes, float** out);

int launch_gemm_v3(const float* A, int64_t lda, int transA, const float* B, int64_t ldb, int transB, float* C,
                   int64_t ldc, int M, int N, int K, const float* bias, int relu, int precision, cudaStream_t stream);

int launch_propagate(const GraphTables* g, const DecisionTables* d, const int8_t* seeds, int64_t batch,
                     int64_t seed_stride, int8_t* slots_out, int64_t slots_stride, int8_t* cand_out,
                     int64_t cand_stride, uint8_t* outcome, int32_t* counts, cudaStream_t stream);

int run_trace(const GraphTables* g, const DecisionTables* d, const int8_t* seeds_host, const int8_t* init_host,
              int8_t* slots_host,
              int32_t* outcome_host, int32_t* site_out, cudaStream_t stream);

}  // namespace apb

struct ap_graph {
  apb::GraphTables t;
};
struct ap_decision {
  apb::DecisionTables t;
};
