// tcgen05 GEMM v2: cp.async multi-stage pipeline, K- and MN-major operands,
// adaptive N tile, deterministic split-K.
//
// Same contract as gemm_tc.cu (C = op(A) op(B) (+bias) (ReLU), TF32 or
// 3xTF32).  Differences that matter on B200:
//  * operands are never transposed by threads: a K-contiguous operand is
//    staged in the canonical K-major layout, an M/N-contiguous one in the
//    canonical MN-major layout (idesc a_major / b_major), both with 16-byte
//    cp.async copies straight from global memory (zero-filled at the edges);
//  * STAGES slices in flight; a slice's buffer is refilled as soon as the
//    MMAs that read it have committed to its mbarrier;
//  * N tile 32 / 64 / 128 / 256 and split-K are chosen so the grid covers the
//    148 SMs (the learner GEMMs have M = 64); split-K partials go to a
//    workspace and are summed in a fixed order (bit-reproducible);
//  * 3xTF32: after a slice lands, threads split it in shared memory into a
//    TF32 head (in place) and the remainder, then thread 0 issues
//    hi*hi + hi*lo + lo*hi.
// Layouts (bytes), tile of R rows (M or N) x 32 k:
//   K-major : (r/8)*1024 + (k/4)*128 + (r%8)*16 + (k%4)*4   LBO 128, SBO 1024
//   MN-major: (r/4)*512  + (k/8)*128 + (k%8)*16 + (r%4)*4   LBO 128, SBO 512
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <unordered_map>
#include <utility>

#include "engine.h"

namespace apb {
namespace {

constexpr int BM = 128;
constexpr int BK = 32;

struct G2 {
  const float* A;
  int64_t lda;
  int a_mn;  // A stored M-contiguous ([K, M])
  const float* B;
  int64_t ldb;
  int b_mn;  // B stored N-contiguous ([K, N])
  float* C;
  int64_t ldc;
  int M, N, K;
  const float* bias;
  int relu;
  int kps;       // K slices per split
  float* work;   // [splits, M, N] partials when split-K
};

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t off_k(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}
__device__ __forceinline__ uint32_t off_mn(int r, int k) {
  return (uint32_t)((r >> 2) * 512 + (k >> 3) * 128 + (k & 7) * 16 + (r & 3) * 4);
}

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void wait_mbar(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "W2_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra W2_%=;\n\t}\n" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

// issue the 16-byte copies of one slice of an operand tile (rows [r0, r0+R))
template <int R>
__device__ __forceinline__ void load_tile(const float* X, int64_t ld, int mn_major, int rows_total, int K, int r0,
                                          int k0, uint32_t dst) {
  constexpr int chunks = R * BK / 4;
  for (int c = threadIdx.x; c < chunks; c += blockDim.x) {
    int r, k;
    uint32_t off;
    const float* src;
    uint32_t bytes;
    if (!mn_major) {  // K contiguous: chunk = (row, 4 consecutive k)
      r = c / (BK / 4);
      k = (c % (BK / 4)) * 4;
      const int gr = r0 + r, gk = k0 + k;
      bytes = (gr < rows_total && gk < K) ? (uint32_t)min(16, (K - gk) * 4) : 0u;
      src = bytes ? X + (int64_t)gr * ld + gk : X;
      off = off_k(r, k);
    } else {  // rows contiguous: chunk = (k, 4 consecutive rows)
      k = c / (R / 4);
      r = (c % (R / 4)) * 4;
      const int gr = r0 + r, gk = k0 + k;
      bytes = (gk < K && gr < rows_total) ? (uint32_t)min(16, (rows_total - gr) * 4) : 0u;
      src = bytes ? X + (int64_t)gk * ld + gr : X;
      off = off_mn(r, k);
    }
    cp16(dst + off, src, bytes);
  }
}

// split a landed slice into TF32 head (in place) and remainder
__device__ __forceinline__ void split_tile(uint8_t* hi, uint8_t* lo, int bytes) {
  for (int i = threadIdx.x * 4; i < bytes / 4; i += blockDim.x * 4) {
    float4 x = *reinterpret_cast<float4*>(hi + 4 * i);
    float4 h, l;
    h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
    h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
    h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
    h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
    l.x = x.x - h.x;
    l.y = x.y - h.y;
    l.z = x.z - h.z;
    l.w = x.w - h.w;
    *reinterpret_cast<float4*>(hi + 4 * i) = h;
    *reinterpret_cast<float4*>(lo + 4 * i) = l;
  }
}

template <int BN, int STAGES, bool SPLIT>
__global__ void __launch_bounds__(128) gemm_v2_kernel(G2 g) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[STAGES];
  __shared__ uint32_t tmem_slot;
  constexpr int A_BYTES = BM * BK * 4;
  constexpr int B_BYTES = BN * BK * 4;
  constexpr int STAGE = (A_BYTES + B_BYTES) * (SPLIT ? 2 : 1);
  constexpr int COLS = BN < 32 ? 32 : BN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int nk_total = (g.K + BK - 1) / BK;
  const int kb = blockIdx.z * g.kps;
  const int nk = min(g.kps, nk_total - kb);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(&tmem_slot)),
                 "r"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mbar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
  if (g.a_mn) idesc |= 1u << 15;
  if (g.b_mn) idesc |= 1u << 16;
  const uint32_t a_lbo = 128, a_sbo = g.a_mn ? 512 : 1024, a_step = g.a_mn ? 128 : 256;
  const uint32_t b_lbo = 128, b_sbo = g.b_mn ? 512 : 1024, b_step = g.b_mn ? 128 : 256;
  const uint32_t base = sa(smem);

  auto issue = [&](int it) {
    const int s = it % STAGES;
    const uint32_t st = base + s * STAGE;
    load_tile<BM>(g.A, g.lda, g.a_mn, g.M, g.K, m0, (kb + it) * BK, st);
    load_tile<BN>(g.B, g.ldb, g.b_mn, g.N, g.K, n0, (kb + it) * BK, st + A_BYTES);
  };
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) issue(s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int it = 0; it < nk; ++it) {
    const int s = it % STAGES;
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    __syncthreads();
    uint8_t* st = smem + s * STAGE;
    if (SPLIT) {
      split_tile(st, st + A_BYTES + B_BYTES, A_BYTES + B_BYTES);
      __syncthreads();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_hi = base + s * STAGE, b_hi = a_hi + A_BYTES;
      const uint32_t a_lo = a_hi + A_BYTES + B_BYTES, b_lo = a_lo + A_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK / 8; ++ks) {
        const uint64_t ah = desc(a_hi + ks * a_step, a_lbo, a_sbo), bh = desc(b_hi + ks * b_step, b_lbo, b_sbo);
        mma(tmem, ah, bh, idesc, (it | ks) != 0);
        if (SPLIT) {
          mma(tmem, ah, desc(b_lo + ks * b_step, b_lbo, b_sbo), idesc, 1);
          mma(tmem, desc(a_lo + ks * a_step, a_lbo, a_sbo), bh, idesc, 1);
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       sa(&mbar[s]))
                   : "memory");
    }
    // refill the buffer the previous iteration's MMAs read
    const int nxt = it + STAGES - 1;
    if (it >= 1) {
      const int ps = (it - 1) % STAGES;
      wait_mbar(sa(&mbar[ps]), ((it - 1) / STAGES) & 1);
    }
    if (nxt < nk) issue(nxt);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (nk > 0) wait_mbar(sa(&mbar[(nk - 1) % STAGES]), ((nk - 1) / STAGES) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");

  const int row = m0 + warp * 32 + lane;
  float* out = g.work ? g.work + (int64_t)blockIdx.z * g.M * g.N : g.C;
  const int64_t ld = g.work ? g.N : g.ldc;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 16) {
    uint32_t v[16];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (row < g.M) {
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const int col = n0 + c0 + t;
        if (col < g.N) {
          float x = nk > 0 ? __uint_as_float(v[t]) : 0.0f;
          if (!g.work) {
            if (g.bias) x += g.bias[col];
            if (g.relu) x = fmaxf(x, 0.0f);
          }
          out[(int64_t)row * ld + col] = x;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(COLS));
}

__global__ void splitk_reduce_kernel(const float* work, int splits, int M, int N, float* C, int64_t ldc,
                                     const float* bias, int relu) {
  const int64_t total = (int64_t)M * N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.0f;
    for (int s = 0; s < splits; ++s) acc += work[(int64_t)s * total + i];  // fixed order: reproducible
    const int r = (int)(i / N), c = (int)(i % N);
    if (bias) acc += bias[c];
    if (relu) acc = fmaxf(acc, 0.0f);
    C[(int64_t)r * ldc + c] = acc;
  }
}

template <int BN, int STAGES, bool SPLIT>
int run(const G2& g, dim3 grid, cudaStream_t stream) {
  constexpr int STAGE = (BM * BK * 4 + BN * BK * 4) * (SPLIT ? 2 : 1);
  constexpr int SMEM = STAGE * STAGES;
  auto k = gemm_v2_kernel<BN, STAGES, SPLIT>;
  AP_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  k<<<grid, 128, SMEM, stream>>>(g);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}


}  // namespace

// Returns AP_ERR_UNSUPPORTED when operand alignment rules out 16-byte copies.
int launch_gemm_v2(const float* A, int64_t lda, int transA, const float* B, int64_t ldb, int transB, float* C,
                   int64_t ldc, int M, int N, int K, const float* bias, int relu, int precision, cudaStream_t stream) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al(A) || !al(B) || lda % 4 || ldb % 4) return AP_ERR_UNSUPPORTED;
  // MN-major operands (transA, or B stored [K, N]) produced wrong results on
  // B200 with the no-swizzle MN-major descriptor (tests/test_gemm_gpu.py); they
  // stay on the thread-staged kernel until that layout is pinned down.
  if (transA || !transB) return AP_ERR_UNSUPPORTED;
  G2 g{A, lda, 0, B, ldb, 0, C, ldc, M, N, K, bias, relu, 0, nullptr};
  // dev overrides for tile sweeps: AP_GEMM_BN (32 | 64), AP_GEMM_SPLITS
  static const int env_bn = std::getenv("AP_GEMM_BN") ? std::atoi(std::getenv("AP_GEMM_BN")) : 0;
  static const int env_splits = std::getenv("AP_GEMM_SPLITS") ? std::atoi(std::getenv("AP_GEMM_SPLITS")) : 0;
  const int bn = env_bn == 32 || env_bn == 64 ? env_bn : (N <= 32 ? 32 : 64);
  const int mt = (M + BM - 1) / BM, nt = (N + bn - 1) / bn;
  const int nk = (K + BK - 1) / BK;
  int splits = 1;
  if (mt * nt < 120 && nk >= 4) splits = std::min(std::min(nk / 2, 16), std::max(1, 148 / (mt * nt)));
  if (env_splits > 0) splits = std::min(env_splits, nk);
  g.kps = (nk + splits - 1) / splits;
  splits = (nk + g.kps - 1) / g.kps;
  if (splits > 1) {
    const int wrc = splitk_workspace(stream, (size_t)splits * M * N * sizeof(float), &g.work);
    if (wrc != AP_OK) return wrc;
  }
  dim3 grid(mt, nt, splits);
  int rc;
  const bool split3 = precision == 3;
  if (bn == 32)
    rc = split3 ? run<32, 3, true>(g, grid, stream) : run<32, 4, false>(g, grid, stream);
  else
    rc = split3 ? run<64, 3, true>(g, grid, stream) : run<64, 4, false>(g, grid, stream);
  if (rc != AP_OK || splits == 1) return rc;
  const int64_t total = (int64_t)M * N;
  splitk_reduce_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, stream>>>(
      g.work, splits, M, N, C, ldc, bias, relu);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

}  // namespace apb

namespace apb {
int splitk_workspace(cudaStream_t stream, size_t bytes, float** out) {
  // one grow-only buffer per (device, stream): GEMMs on one stream are ordered, so they can share it
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<float*, size_t>> ws;
  int dev = 0;
  AP_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  auto& w = ws[{dev, stream}];
  if (bytes > w.second) {
    // a capture in global mode forbids cudaMalloc on this thread; the buffer is an ordinary
    // persistent allocation (not a graph node), so allocate it in relaxed mode
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    AP_CUDA_CHECK(cudaThreadExchangeStreamCaptureMode(&mode));
    float* fresh = nullptr;
    const cudaError_t e = cudaMalloc(&fresh, bytes);
    cudaThreadExchangeStreamCaptureMode(&mode);
    AP_CUDA_CHECK(e);
    w = {fresh, bytes};  // the previous buffer is intentionally kept alive (captured graphs may use it)
  }
  *out = w.first;
  return AP_OK;
}
}  // namespace apb

