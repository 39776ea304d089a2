// tcgen05 GEMM v3: TMA-fed, warp-specialised, 128-byte swizzle (TF32, K-major).
//
// C[M, N] = A[M, K] * B[N, K]^T (+ bias[N]) (ReLU), fp32 in / fp32 out, TF32
// tensor-core math (the throughput-mode Q-network GEMMs; 3xTF32 stays on v2).
//   * operand tiles are moved by TMA (cp.async.bulk.tensor.2d) with
//     CU_TENSOR_MAP_SWIZZLE_128B: box = 32 fp32 (one 128-byte row) x rows, which
//     is exactly the canonical K-major SW128 UMMA atom (8 rows x 128 B, SBO 1024);
//     out-of-bounds rows / k are zero-filled by the TMA unit;
//   * a STAGES-deep ring with full (TMA complete_tx) and empty (tcgen05.commit)
//     mbarriers: thread 0 of warp 0 produces, thread 0 of warp 1 issues the
//     MMAs (4 x K=8 per 32-wide k slice, the descriptor start advanced by 32 B
//     inside the swizzled row), accumulators in TMEM;
//   * epilogue: all 4 warps tcgen05.ld their 32 TMEM lanes into a [128][BN+1]
//     shared tile (the drained stage ring), then each thread owns one column
//     (bias loaded once) and consecutive threads store consecutive columns;
//   * split-K (only when K >= 512 and the tile grid leaves SMs idle): the splits
//     of a tile form one thread-block cluster (<= 16 CTAs) and reduce through
//     DSMEM in split order (bit-reproducible); AP_GEMM_NO_CLUSTER=1 uses a
//     per-stream global workspace + a fixed-order reduce kernel instead;
//   * BN = 32 | 64 | 128 (128 when it needs fewer waves than 64);
//   * programmatic dependent launch: the TMEM / barrier / tensor-map prologue
//     overlaps the previous kernel (griddepcontrol.wait before any global access).
// Tensor maps are encoded per call with cuTensorMapEncodeTiled obtained through
// cudaGetDriverEntryPoint (no libcuda link dependency).
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "engine.h"

namespace apb {
namespace {

constexpr int BM3 = 128;
constexpr int BK3 = 32;  // fp32 elements = 128 bytes = one swizzle row

struct G3 {
  float* C;
  int64_t ldc;
  int M, N, K;
  const float* bias;
  int relu;
  int kps;      // k slices per split
  float* work;  // [splits, M, N] partials when split-K through global memory
  int cluster;  // split-K CTAs of a tile form one cluster: reduce through DSMEM
  // fused Adam epilogue (am != nullptr; unsplit GEMMs only): C is a weight gradient,
  // am / av / ap the Adam moments and parameters at C's offset (same layout, ld = ldc)
  float *am, *av, *ap;
  const int64_t* actl;
  float lr, b1, b2, eps;
  int t_add;       // Adam step t = ctl[AP_CTL_TRAIN] + t_add
  float* tdst;     // transposed parameter copy tdst[c][r] for rows r < trows
  int64_t tld;
  int trows;
};

__device__ __forceinline__ uint32_t sa3(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  // start >> 4 | LBO field 1 (unused for swizzled K-major) | SBO 1024 B >> 4 |
  // version 1 (bit 46) | layout SWIZZLE_128B (2 at bits 61-63)
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "W3_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra W3_%=;\n\t}\n" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(map), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}

#ifdef AP_GEMM_TRACE  // dev-only: SM-clock stamps of CTA (0,0,0) (scratch/gemm_trace)
__device__ long long g_trace[8];
#define GTRACE(k)                                                                   \
  do {                                                                              \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0) g_trace[k] = clock64(); \
  } while (0)
#else
#define GTRACE(k) \
  do {            \
  } while (0)
#endif

template <int BN, int STAGES>
__global__ void __launch_bounds__(128) gemm_v3_kernel(const __grid_constant__ CUtensorMap tmA,
                                                      const __grid_constant__ CUtensorMap tmB, G3 g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t tmem_slot;
  constexpr int A_BYTES = BM3 * BK3 * 4;
  constexpr int B_BYTES = BN * BK3 * 4;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int COLS = BN < 32 ? 32 : BN;
  // 1024-byte aligned stage base (SWIZZLE_128B atoms)
  const uint32_t base = (sa3(smem_raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM3, n0 = blockIdx.y * BN;
  const int nk_total = (g.K + BK3 - 1) / BK3;
  const int kb = blockIdx.z * g.kps;
  const int nk = max(0, min(g.kps, nk_total - kb));

  if (threadIdx.x == 0) GTRACE(0);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa3(&tmem_slot)),
                 "r"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa3(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa3(&empty[s])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa3(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;
  if (threadIdx.x == 0) GTRACE(1);
  // PDL: the TMEM / barrier / tensor-map prologue above overlapped the previous
  // kernel; no global memory is touched before its writes are visible
  pdl_trigger();
  pdl_wait();

  if (threadIdx.x == 0) {
    // TMA producer
    for (int it = 0; it < nk; ++it) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(sa3(&empty[s]), ((it / STAGES) - 1) & 1);
      const uint32_t st = base + s * STAGE;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa3(&full[s])), "r"(STAGE)
                   : "memory");
      const int kc = (kb + it) * BK3;
      tma_load_2d(st, &tmA, kc, m0, sa3(&full[s]));
      tma_load_2d(st + A_BYTES, &tmB, kc, n0, sa3(&full[s]));
    }
  } else if (threadIdx.x == 32) {
    // MMA issuer
    const uint32_t idesc =
        (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM3 >> 4) << 24);
    for (int it = 0; it < nk; ++it) {
      const int s = it % STAGES;
      mbar_wait(sa3(&full[s]), (it / STAGES) & 1);
      if (it == 0) GTRACE(2);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a = base + s * STAGE, b = a + A_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK3 / 8; ++ks) {
        const uint64_t da = desc_sw128(a + ks * 32), db = desc_sw128(b + ks * 32);
        const uint32_t acc = (it | ks) != 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       sa3(&empty[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa3(&done))
                 : "memory");
  }
  __syncwarp();
  if (nk > 0) mbar_wait(sa3(&done), 0);
  if (threadIdx.x == 0) GTRACE(3);
  asm volatile("tcgen05.fence::after_thread_sync;");

  if (g.cluster) {
    // split-K through distributed shared memory: every CTA of the cluster (the
    // splits of one output tile) parks its partial tile in its own shared
    // memory (the drained stage ring, rows padded to BN + 1 floats), then CTA
    // r sums row slice r over all splits in split order and stores C
    constexpr int LDP = BN + 1;
    float* part = reinterpret_cast<float*>(smem_raw + (base - sa3(smem_raw)));
    const int lrow = warp * 32 + lane;
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
#pragma unroll
      for (int t = 0; t < 16; ++t) part[lrow * LDP + c0 + t] = nk > 0 ? __uint_as_float(v[t]) : 0.0f;
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const int S = (int)gridDim.z, rank = (int)blockIdx.z;
    const int vrows = min(BM3, g.M - m0);  // only the tile's valid rows are reduced
    const int rows_per = (vrows + S - 1) / S;
    const int r_lo = rank * rows_per, r_hi = min(vrows, r_lo + rows_per);
    const uint32_t local = sa3(part);
    const int cc = threadIdx.x % BN;  // BN | 128: one column per thread, bias loaded once
    const float bcc = (g.bias && n0 + cc < g.N) ? g.bias[n0 + cc] : 0.0f;
    for (int e = threadIdx.x; e < (r_hi - r_lo) * BN; e += blockDim.x) {
      const int r = r_lo + e / BN, c = cc;
      const int grow = m0 + r, gcol = n0 + c;
      if (grow >= g.M || gcol >= g.N) continue;
      const uint32_t off = local + (uint32_t)(r * LDP + c) * 4u;
      // all splits' loads in flight first, then the sum in split order
      float x[16];
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        x[s] = 0.0f;
        if (s < S) {
          uint32_t ra;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(off), "r"(s));
          asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x[s]) : "r"(ra));
        }
      }
      float acc = 0.0f;
#pragma unroll
      for (int s = 0; s < 16; ++s)
        if (s < S) acc += x[s];
      if (g.bias) acc += bcc;
      if (g.relu) acc = fmaxf(acc, 0.0f);
      g.C[(int64_t)grow * g.ldc + gcol] = acc;
    }
    if (threadIdx.x == 0) GTRACE(4);
    // no CTA may leave while a peer still reads its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(COLS));
    if (threadIdx.x == 0) GTRACE(5);
    return;
  }

  // Epilogue through shared memory: TMEM rows (one per lane) go into the
  // drained stage ring ([BM][BN+1], conflict-free), then consecutive threads
  // store consecutive columns of a row -- one transaction per warp store
  // instead of 32 (a lane-per-row store was ~4 us of a small GEMM).
  float* out = g.work ? g.work + (int64_t)blockIdx.z * g.M * g.N : g.C;
  const int64_t ld = g.work ? g.N : g.ldc;
  constexpr int LDT = BN + 1;
  float* tile = reinterpret_cast<float*>(smem_raw + (base - sa3(smem_raw)));
  const int lrow = warp * 32 + lane;
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
#pragma unroll
    for (int t = 0; t < 16; ++t) tile[lrow * LDT + c0 + t] = nk > 0 ? __uint_as_float(v[t]) : 0.0f;
  }
  __syncthreads();
  // 128 threads, BN | 128: each thread owns one column (bias loaded once) and
  // walks rows; nothing in the loop waits on a global load
  const int rows = min(BM3, g.M - m0), cols = min(BN, g.N - n0);
  const int c = threadIdx.x % BN;
  if (g.am) {
    // fused Adam: store the gradient, update moments and parameters in place,
    // then write the transposed parameter copy from the tile (coalesced rows)
    __shared__ float s_ic[2];
    if (threadIdx.x == 0) {
      const double t = (double)(g.actl[AP_CTL_TRAIN] + g.t_add);
      s_ic[0] = (float)(1.0 / (1.0 - pow((double)g.b1, t)));
      s_ic[1] = (float)(1.0 / (1.0 - pow((double)g.b2, t)));
    }
    __syncthreads();
    const float ic1 = s_ic[0], ic2 = s_ic[1];
    if (c < cols) {
      constexpr int RS = 128 / BN, D = 8;  // row stride per thread; 8 rows' loads in flight
      float* __restrict__ am = g.am;
      float* __restrict__ av = g.av;
      float* __restrict__ ap = g.ap;
      for (int r0 = threadIdx.x / BN; r0 < rows; r0 += D * RS) {
        float mi[D], vi[D], pi[D];
#pragma unroll
        for (int u = 0; u < D; ++u) {
          const int r = r0 + u * RS;
          if (r < rows) {
            const int64_t i = (int64_t)(m0 + r) * ld + n0 + c;
            mi[u] = am[i];
            vi[u] = av[i];
            pi[u] = ap[i];
          }
        }
#pragma unroll
        for (int u = 0; u < D; ++u) {
          const int r = r0 + u * RS;
          if (r < rows) {
            const int64_t i = (int64_t)(m0 + r) * ld + n0 + c;
            const float gr = tile[r * LDT + c];
            out[i] = gr;
            adam_math(gr, mi[u], vi[u], pi[u], g.lr, g.b1, g.b2, g.eps, ic1, ic2);
            am[i] = mi[u];
            av[i] = vi[u];
            ap[i] = pi[u];
            tile[r * LDT + c] = pi[u];
          }
        }
      }
    }
    __syncthreads();
    const int trr = min(rows, g.trows - m0);
    if (g.tdst && trr > 0)
      for (int e = threadIdx.x; e < cols * trr; e += blockDim.x) {
        const int cc = e / trr, rr = e % trr;
        g.tdst[(int64_t)(n0 + cc) * g.tld + m0 + rr] = tile[rr * LDT + cc];
      }
  } else if (c < cols) {
    const bool epi = !g.work;
    const bool has_bias = epi && g.bias;
    const float bc = has_bias ? g.bias[n0 + c] : 0.0f;
    const bool relu = epi && g.relu;
    float* __restrict__ o = out + (int64_t)m0 * ld + n0 + c;
#pragma unroll 4
    for (int r = threadIdx.x / BN; r < rows; r += 128 / BN) {
      float x = tile[r * LDT + c];
      if (has_bias) x += bc;
      if (relu) x = fmaxf(x, 0.0f);
      o[(int64_t)r * ld] = x;
    }
  }
  if (threadIdx.x == 0) GTRACE(4);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(COLS));
  if (threadIdx.x == 0) GTRACE(5);
}

// A-tile multicast variant (unsplit grids, plain bias / ReLU epilogue): the MC
// CTAs of a cluster share an M tile and take consecutive N tiles; each loads a
// 1/MC slice of the A tile and multicasts it to every CTA of the cluster, so
// A is read once per cluster instead of once per CTA.  A stage is released
// when all MC consumers have committed (empty barriers count MC, every MMA
// commit arrives on the whole cluster).
template <int BN, int STAGES, int MC>
__global__ void __launch_bounds__(128) gemm_v3_mc_kernel(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB, G3 g) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], done;
  __shared__ uint32_t tmem_slot;
  constexpr int A_BYTES = BM3 * BK3 * 4;
  constexpr int B_BYTES = BN * BK3 * 4;
  constexpr int STAGE = A_BYTES + B_BYTES;
  constexpr int AQ = A_BYTES / MC;  // one CTA's slice of the A tile (BM3 / MC rows)
  constexpr uint16_t kMask = (uint16_t)((1u << MC) - 1u);
  const uint32_t base = (sa3(smem_raw) + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM3, n0 = blockIdx.y * BN;
  const int nk = (g.K + BK3 - 1) / BK3;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa3(&tmem_slot)), "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < STAGES; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa3(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa3(&empty[s])), "r"(MC));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa3(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // every barrier of the cluster is initialised before any multicast can reach it
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (threadIdx.x == 0) {
    for (int it = 0; it < nk; ++it) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(sa3(&empty[s]), ((it / STAGES) - 1) & 1);
      const uint32_t st = base + s * STAGE;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa3(&full[s])), "r"(STAGE)
                   : "memory");
      const int kc = it * BK3;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
          " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(st + rank * AQ),
          "l"(&tmA), "r"(kc), "r"(m0 + (int)rank * (BM3 / MC)), "r"(sa3(&full[s])), "h"(kMask)
          : "memory");
      tma_load_2d(st + A_BYTES, &tmB, kc, n0, sa3(&full[s]));
    }
  } else if (threadIdx.x == 32) {
    const uint32_t idesc =
        (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM3 >> 4) << 24);
    for (int it = 0; it < nk; ++it) {
      const int s = it % STAGES;
      mbar_wait(sa3(&full[s]), (it / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a = base + s * STAGE, b = a + A_BYTES;
#pragma unroll
      for (int ks = 0; ks < BK3 / 8; ++ks) {
        const uint64_t da = desc_sw128(a + ks * 32), db = desc_sw128(b + ks * 32);
        const uint32_t acc = (it | ks) != 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              sa3(&empty[s])),
          "h"(kMask)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa3(&done))
                 : "memory");
  }
  __syncwarp();
  if (nk > 0) mbar_wait(sa3(&done), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: as gemm_v3_kernel (staged tile, one column per thread)
  constexpr int LDT = BN + 1;
  float* tile = reinterpret_cast<float*>(smem_raw + (base - sa3(smem_raw)));
  const int lrow = warp * 32 + lane;
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
#pragma unroll
    for (int t = 0; t < 16; ++t) tile[lrow * LDT + c0 + t] = nk > 0 ? __uint_as_float(v[t]) : 0.0f;
  }
  __syncthreads();
  const int rows = min(BM3, g.M - m0), cols = min(BN, g.N - n0);
  const int c = threadIdx.x % BN;
  if (c < cols) {
    const float bc = g.bias ? g.bias[n0 + c] : 0.0f;
    float* __restrict__ o = g.C + (int64_t)m0 * g.ldc + n0 + c;
#pragma unroll 4
    for (int r = threadIdx.x / BN; r < rows; r += 128 / BN) {
      float x = tile[r * LDT + c];
      if (g.bias) x += bc;
      if (g.relu) x = fmaxf(x, 0.0f);
      o[(int64_t)r * g.ldc] = x;
    }
  }
  // no CTA may exit while a peer's multicast commit can still arrive on its barriers
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
}

__global__ void splitk_reduce3_kernel(const float* work, int splits, int M, int N, float* C, int64_t ldc,
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

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  // driver entry points are process-wide; a function-local static initialises once, thread-safely
  static const EncodeTiled fn = []() -> EncodeTiled {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiled>(p);
    return nullptr;
  }();
  return fn;
}

// row-major [rows, K] fp32 (K contiguous, ld elements), box 32 x box_rows, SW128
bool make_map(CUtensorMap* m, const float* ptr, int64_t rows, int64_t K, int64_t ld, int box_rows) {
  EncodeTiled fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)BK3, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int STAGES>
int run3(const CUtensorMap& ma, const CUtensorMap& mb, const G3& g, dim3 grid, cudaStream_t s) {
  constexpr int SMEM = (BM3 + BN) * BK3 * 4 * STAGES + 1024;
  auto k = gemm_v3_kernel<BN, STAGES>;
  static PerDeviceMax configured;
  if (configured.need(current_device(), 1)) {
    AP_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    // split-K clusters of up to 16 CTAs (beyond the portable 8)
    AP_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
  if (!g.cluster) {
    launch_pdl(k, grid, dim3(128), SMEM, s, ma, mb, g);
    AP_CUDA_CHECK(cudaGetLastError());
    return AP_OK;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = grid.z;  // the split-K CTAs of one tile
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  AP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k, ma, mb, g));
  return AP_OK;
}


}  // namespace

// TF32 only, both operands K-major (A [M, K], B [N, K]); AP_ERR_UNSUPPORTED otherwise.
static int launch_v3_impl(const float* A, int64_t lda, int transA, const float* B, int64_t ldb, int transB, float* C,
                          int64_t ldc, int M, int N, int K, const float* bias, int relu, int precision,
                          cudaStream_t stream, const G3* adam);

int launch_gemm_v3(const float* A, int64_t lda, int transA, const float* B, int64_t ldb, int transB, float* C,
                   int64_t ldc, int M, int N, int K, const float* bias, int relu, int precision, cudaStream_t stream) {
  return launch_v3_impl(A, lda, transA, B, ldb, transB, C, ldc, M, N, K, bias, relu, precision, stream, nullptr);
}

static int launch_v3_impl(const float* A, int64_t lda, int transA, const float* B, int64_t ldb, int transB, float* C,
                          int64_t ldc, int M, int N, int K, const float* bias, int relu, int precision,
                          cudaStream_t stream, const G3* adam) {
  if (precision != 1 || transA || !transB || std::getenv("AP_GEMM_NO_TMA")) return AP_ERR_UNSUPPORTED;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!al(A) || !al(B) || lda % 4 || ldb % 4 || M < 1 || N < 1 || K < 1) return AP_ERR_UNSUPPORTED;
  // BN: 32 for narrow N; 128 when the BN=64 grid (one CTA per SM) needs more waves over the 148 SMs
  // than the BN=128 grid (measured: 12681x64x256 12.5 -> 9.4 us, 1024x256x3171 16.7 -> 12.4 us,
  // 257x64x3171 7.2 -> 5.3 us; grids that fit one wave either way stay at 64).  AP_GEMM_V3_BN=64|128 forces.
  const int env_bn = std::getenv("AP_GEMM_V3_BN") ? std::atoi(std::getenv("AP_GEMM_V3_BN")) : 0;
  int bn = (N <= 32 || env_bn == 32) ? 32 : 64;
  if (bn == 64 && N > 64) {
    const int64_t mt0 = (M + BM3 - 1) / BM3;
    const int64_t w64 = (mt0 * ((N + 63) / 64) + 147) / 148, w128 = (mt0 * ((N + 127) / 128) + 147) / 148;
    const bool unsplit = mt0 * ((N + 63) / 64) >= 120;
    if (env_bn == 128 || (env_bn == 0 && unsplit && w128 < w64)) bn = 128;
  }
  CUtensorMap ma, mb;
  if (!make_map(&ma, A, M, K, lda, BM3) || !make_map(&mb, B, N, K, ldb, bn)) return AP_ERR_UNSUPPORTED;
  G3 g{C, ldc, M, N, K, bias, relu, 0, nullptr, 0};
  if (adam) {  // the Adam fields; bias / ReLU do not apply to a gradient
    g = *adam;
    g.C = C, g.ldc = ldc, g.M = M, g.N = N, g.K = K, g.bias = nullptr, g.relu = 0, g.kps = 0, g.work = nullptr;
    g.cluster = 0;
  }
  const int mt = (M + BM3 - 1) / BM3, nt = (N + bn - 1) / bn;
  const int nk = (K + BK3 - 1) / BK3;
  // split-K for grids that would leave SMs idle; the splits of a tile reduce
  // inside one thread-block cluster (<= 16 CTAs, non-portable size) through
  // DSMEM: no workspace, no extra launch (AP_GEMM_NO_CLUSTER=1: workspace path)
  const bool no_cluster = std::getenv("AP_GEMM_NO_CLUSTER") != nullptr;
  const int max_split = std::getenv("AP_GEMM_MAX_SPLIT") ? std::atoi(std::getenv("AP_GEMM_MAX_SPLIT")) : 16;
  int splits = 1;
  // (measured on B200 with the staged epilogue: a split costs a cluster barrier pair and a DSMEM
  // reduce, ~2-3 us, which only pays once each split saves several k slices -- K >= 512)
  if (mt * nt < 120 && nk >= 16) splits = std::min(std::min(nk / 2, max_split), std::max(1, 148 / (mt * nt)));
  // dev knobs for sweeps: AP_GEMM_V3_SPLITS (forced split count), AP_GEMM_V3_STAGES (4 | 6)
  if (const char* e = std::getenv("AP_GEMM_V3_SPLITS")) splits = std::max(1, std::min(std::atoi(e), nk));
  const int env_stages = std::getenv("AP_GEMM_V3_STAGES") ? std::atoi(std::getenv("AP_GEMM_V3_STAGES")) : 0;
  const bool four_stages = env_stages == 4, eight_stages = env_stages == 8 && bn == 64;
  g.kps = (nk + splits - 1) / splits;
  splits = (nk + g.kps - 1) / g.kps;
  if (adam && splits > 1) return AP_ERR_UNSUPPORTED;  // the fused epilogue needs the whole gradient tile
  if (splits > 1 && splits <= 16 && !no_cluster) g.cluster = 1;
  if (splits > 1 && !g.cluster) {
    const int wrc = splitk_workspace(stream, (size_t)splits * M * N * sizeof(float), &g.work);
    if (wrc != AP_OK) return wrc;
  }
  const dim3 grid(mt, nt, splits);
  // A-tile multicast across 4 N tiles of a cluster for unsplit grids with K >= 512 (measured on B200:
  // 4096x1060x256 14.3 -> 12.7 us; at K = 256 the cluster syncs cost more than the saved A reads, 5.6 -> 6.3 us).
  // AP_GEMM_NO_MC=1 disables it, AP_GEMM_MC=1 forces it for any eligible shape.
  const bool use_mc = !std::getenv("AP_GEMM_NO_MC") && (std::getenv("AP_GEMM_MC") || nk >= 16);
  if (!adam && splits == 1 && bn == 64 && nt % 4 == 0 && use_mc) {
    CUtensorMap maq;
    if (!make_map(&maq, A, M, K, lda, BM3 / 4)) return AP_ERR_UNSUPPORTED;
    // stages in flight: the kernel is bound by the L2 -> shared-memory ingest of its operand
    // tiles (24 KB per k slice); AP_GEMM_MC_STAGES = 6 | 8 (sweep knob)
    const int mc_stages = std::getenv("AP_GEMM_MC_STAGES") ? std::atoi(std::getenv("AP_GEMM_MC_STAGES")) : 6;
    const int SMEM = (BM3 + 64) * BK3 * 4 * (mc_stages == 8 ? 8 : 6) + 1024;
    auto k = mc_stages == 8 ? gemm_v3_mc_kernel<64, 8, 4> : gemm_v3_mc_kernel<64, 6, 4>;
    static PerDeviceMax mc_configured;
    if (mc_configured.need(current_device(), SMEM))
      AP_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 4;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    AP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k, maq, mb, g));
    return AP_OK;
  }
  const int rc = bn == 128     ? run3<128, 6>(ma, mb, g, grid, stream)
                 : eight_stages ? run3<64, 8>(ma, mb, g, grid, stream)
                 : four_stages ? (bn == 32 ? run3<32, 4>(ma, mb, g, grid, stream) : run3<64, 4>(ma, mb, g, grid, stream))
                               : (bn == 32 ? run3<32, 6>(ma, mb, g, grid, stream) : run3<64, 6>(ma, mb, g, grid, stream));
  if (rc != AP_OK || splits == 1 || g.cluster) return rc;
  const int64_t total = (int64_t)M * N;
  splitk_reduce3_kernel<<<(int)std::min<int64_t>((total + 255) / 256, 148 * 8), 256, 0, stream>>>(
      g.work, splits, M, N, C, ldc, bias, relu);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

}  // namespace apb

#ifdef AP_GEMM_TRACE
extern "C" int ap_gemm_trace_read(long long* out) {
  return cudaMemcpyFromSymbol(out, apb::g_trace, sizeof(long long) * 8) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" int ap_gemm_tf32_adam(const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                                 int32_t M, int32_t N, int32_t K, float* m, float* v, float* params,
                                 const int64_t* ctl, int32_t counter_advanced, float lr, float beta1, float beta2,
                                 float eps, float* t_dst, int64_t t_ld, int32_t t_rows, void* stream) {
  if (!A || !B || !C || !m || !v || !params || !ctl || M < 1 || N < 1 || K < 1 || (t_dst && t_ld < t_rows)) {
    apb::set_error("ap_gemm_tf32_adam: bad arguments");
    return AP_ERR_INVALID;
  }
  apb::G3 a{};
  a.am = m, a.av = v, a.ap = params, a.actl = ctl;
  a.lr = lr, a.b1 = beta1, a.b2 = beta2, a.eps = eps, a.t_add = counter_advanced ? 0 : 1;
  a.tdst = t_dst, a.tld = t_ld, a.trows = t_dst ? t_rows : 0;
  return apb::launch_v3_impl(A, lda, 0, B, ldb, 1, C, ldc, M, N, K, nullptr, 0, 1, (cudaStream_t)stream, &a);
}
