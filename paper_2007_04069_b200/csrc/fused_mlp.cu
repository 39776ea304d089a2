// Fused dueling-MLP learner and forward for small batches (the parity agent and
// the device search loop): one persistent kernel per DQN learn step.
//
// The reference learner (agent.py:258-299) at its batch of 64 is three small
// forwards (online and target on the next states, online on the states), a
// double-DQN TD with Huber and importance weights, the analytic backward of a
// dueling MLP and Adam.  As separate tensor-core GEMMs that is ~40 dependent
// launches of 4-11 us each; here every phase is a set of register-tiled fp32
// tiles spread over all SMs, with grid-wide barriers between dependent phases
// (2L + 2 for L hidden layers, one more for heads wider than 8), so one launch does
// the whole step:
//
//   fwd layer i   H_i = relu(H_{i-1} W_i + b_i)   online rows [next; cur], target rows next
//                 (layer 0 reads the replay-ring rows through the sampled indices)
//   head + TD     z = H_L Wh + bh, Q = V + A - mean(A), double-DQN target, Huber,
//                 dz = dLoss/dz, td, loss terms, priorities |td| + 1e-6 (last duplicate
//                 wins); one warp per sample, small heads computed in its registers
//   head bwd      gWh = H_L^T dz, gbh = colsum dz, dh_L = relu'(H_L) (dz Wh^T)
//   layer i bwd   gW_i = H_{i-1}^T dh_i, gb_i = colsum dh_i, dh_{i-1} = relu'(H_{i-1}) (dh_i W_i^T)
//   Adam          in the epilogue of each weight-gradient tile (a tile sums the whole
//                 batch, so its gradient is final); the transposed copies the dgrads and
//                 the tensor-core forward read are refreshed one phase later
//
// Tile shapes are planned per phase against a fixed 148-SM reference grid, every sum
// runs in a fixed order (k ascending inside a K-group, groups added in order, tiles
// never split K across CTAs), so results are deterministic and independent of the
// launch grid.  fp32 products and sums (FMA) track the fp64 reference to ~1e-6
// relative (tests/test_fused_mlp_gpu.py).  Control state (jobs, workspace pointers)
// lives in shared memory, not in per-thread stacks.  The same kernel in forward mode
// gives Q for a few rows (the act of the search loop).
#include <algorithm>
#include <cstdint>

#include "engine.h"
#include "parity_act.cuh"

namespace apb {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxLayers = 4;  // hidden layers
constexpr int kTN = 32;        // tile columns (one per lane)
constexpr int kSmemFloats = 56 * 1024;  // 224 KB of dynamic shared memory per CTA (one chunk at K <= 1100)

struct Learn;


__device__ __forceinline__ void trace_mark(unsigned long long* tr, int& k) {
  if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[k] = t;
  }
  ++k;
}

#ifdef AP_FUSED_TILE_TRACE  // dev-only: stamps of CTA 0's tiles into trace[4096 + 8 n + k]
__device__ unsigned long long* g_tile_trace;
__device__ int g_tile_n;
#define TT(k)                                                                     \
  do {                                                                            \
    if (blockIdx.x == 0 && threadIdx.x == 0 && g_tile_trace && g_tile_n < 64) {    \
      unsigned long long t_;                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                      \
      g_tile_trace[4096 + 8 * g_tile_n + k] = t_;                                 \
      if (k == 5) ++g_tile_n;                                                     \
    }                                                                             \
  } while (0)
#else
#define TT(k) \
  do {        \
  } while (0)
#endif

// trace mode: each CTA's arrival time at the end of phase k (its work done), after the
// per-phase marks of CTA 0 (tr[64 + k * grid + cta])
__device__ __forceinline__ void trace_arrive(unsigned long long* tr, int k) {
  if (!tr) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[64 + k * gridDim.x + blockIdx.x] = t;
  }
}

// grid-wide barrier (all CTAs co-resident: cooperative launch).  The counter word counts arrivals
// monotonically (it stays a multiple of the grid size between launches, so each word of the
// barrier buffer serves one grid size: word 0 the full-grid phases, words 2 / 3 the few-row
// forward on the full grid / with one SM left free): one release add per CTA, then
// relaxed loads until the count reaches the next multiple.  The CTA barrier before the add
// orders every thread's writes before thread 0's release (cumulativity).
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    const unsigned target = (old / gridDim.x + 1) * gridDim.x;
    unsigned cur;
    // relaxed polls: an acquire load invalidates the SM's L1 on every poll (CCTL.IVALL), which
    // also evicts the CTA's stack; every cross-CTA operand of this kernel is read at L2
    // (ld.global.cg / cp.async.cg), where the releasing CTAs' writes already are
    do {
      asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
    } while ((int)(cur - target) < 0);
  }
  __syncthreads();
}

// A operand of a tile job: element (m, k).  Rows come from `p` with row stride `sr`,
// or from replay-ring rows through the sampled indices (rows [0, split) from p0,
// [split, 2 split) from p1).  trans: element (m, k) lives in row k, column m.
struct AOp {
  const float* p;
  int64_t sr;
  const float* p0;
  const float* p1;
  const int32_t* idx;
  int split;
  int trans;
  int ones_at;  // trans only: row m == ones_at reads 1.0 (bias gradient as one more output row), -1 none
  __host__ __device__ __forceinline__ const float* row(int r) const {
    if (!idx) return p + (int64_t)r * sr;
    return r < split ? p0 + (int64_t)idx[r] * sr : p1 + (int64_t)idx[r - split] * sr;
  }
};

// B operand: element (k, n) at p[k * sk + n * sn]
struct BOp {
  const float* p;
  int64_t sk, sn;
};

// One tiled product C[M, N] = epi(sum_k A(m, k) B(k, n) + bias[n]); epi: relu (1),
// relu' mask from `mask` rows (2), none (0).  Tiles of (8 / kg) * rpt rows x 32 columns:
// lane = column, the 8 warps split into 8 / kg row groups x kg K-groups (partial sums
// added in group order through shared memory, so every sum has one fixed order).
struct Job {
  AOp a;
  BOp b;
  float* c;
  int64_t ldc;
  int M, N, K, rpt, kg;
  const float* bias;
  int epi;
  const float* mask;
  int64_t ldmask;
  // Adam epilogue (weight-gradient jobs, which sum the whole batch inside one tile): C is
  // the gradient block of the parameters at flat offset `eoff`; the tile also applies Adam
  // to them and, with `wt`, writes rows < wt_rows of the transposed copy
  int adam;
  int64_t eoff;
  float* wt;
  int64_t wt_ld;
  int wt_rows;
  __host__ __device__ __forceinline__ int tm() const { return (kWarps / kg) * rpt; }
  __host__ __device__ __forceinline__ int tiles() const { return ((M + tm() - 1) / tm()) * ((N + kTN - 1) / kTN); }
};

static_assert(sizeof(Job) % 4 == 0, "jobs are copied as 32-bit words");
constexpr int kMaxPhases = 2 * kMaxLayers + 2;  // L forwards, wide head, head backward, L backwards

struct Phase {
  Job jobs[3];
  int nj;
};

struct Learn {
  int L, A, B, rows_fwd;  // rows_fwd: forward mode row count (learn mode: 0)
  int d[kMaxLayers + 2];  // d[0] state dim, d[1..L] hidden widths, d[L+1] = 1 + A
  float* p;               // online flat parameters (updated in place)
  const float* tp;        // target flat parameters
  int64_t w_off[kMaxLayers + 1], b_off[kMaxLayers + 1];
  // replay ring and PER sample
  const float* r_states;
  const float* r_next;
  int64_t r_ld;
  const int32_t* r_actions;
  const float* r_rewards;
  const uint8_t* r_done;
  const uint8_t* r_mask;
  double* r_prio;
  const int32_t* idx;
  const float* isw;
  float gamma, delta;
  // Adam
  float* grad;
  float* m;
  float* v;
  int64_t nparams;
  float lr, b1, b2, eps, c1, c2;
  const float* ctab;  // optional bias-correction table (parity loop), see ap_dqn_adam_tab
  const int64_t* ctl;
  int64_t t_offset;
  float* wt[kMaxLayers + 1];  // transposed copies [d_{i+1}, ld] of w_i (and the head)
  int64_t wt_ld[kMaxLayers + 1];
  // outputs
  float* td;
  float* loss;  // sum_b w_b * huber_b
  float* q_out;  // forward mode: [rows, A]
  const float* x_in;  // forward mode: [rows, x_ld]
  int64_t x_ld;
  // workspace
  float* ws;
  unsigned* bar;
  unsigned long long* trace;  // optional: %globaltimer after each phase (CTA 0)
  // planned on the host (plan_phases): every phase's tile jobs and the workspace carve-up
  Phase ph[kMaxPhases];
  int nph;
  float* Hon[kMaxLayers + 1];
  float* Htg[kMaxLayers + 1];
  float* dh[kMaxLayers + 1];
  float *zon, *ztg, *dz, *lrow;
  int64_t gate;               // > 0: no-op while ctl[AP_CTL_SIZE] < gate (self-gated loop body)
  // forward mode, parity loop: the epsilon-greedy act on row 0's Q (parity_act.cuh)
  int act;
  ap_parity_loop pl;
  int32_t* action;
  // parity-loop tail: loss log, train counter, target sync (see ap_fused_learn)
  int64_t* tail_ctl;
  float* loss_log;
  int64_t loss_cap;
  int sync_every, sync_n;
  const float* sync_src[6];
  float* sync_dst[6];
  int64_t sync_count[6];
  int lazy_wt0;              // the first layer's transposed copy is refreshed by the caller
  int reserve;               // SMs the launch leaves free (the few-row forward's barrier word)
  double* r_scaled;          // optional: priorities ** alpha, updated with each priority
  double* pstat;             // with r_scaled: the ring's max priority after the update, its ** alpha
  double alpha;
  const uint64_t* rng_from;  // parity loop, early PER sample: the stream state to commit
  uint64_t* rng_to;
};

__device__ __forceinline__ void cp_async16(float* smem_dst, const float* gsrc) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ bool al16(const float* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

constexpr int kBS = kTN + 4;  // B tile row stride (floats): 16-byte rows, conflict-free column reads

// One tile of a job: rows [m0, m0 + 8 RPT), columns [n0, n0 + 32).  Operands are staged in
// shared memory with cp.async (16-byte asynchronous copies, hundreds in flight per thread)
// where rows are contiguous and aligned, element loads otherwise:
//   A row-major      As[r][k]   (TRANS = 0: contiguous along k)
//   A transposed     At[k][r]   (TRANS = 1: element (m, k) in source row k, contiguous along m)
//   B                Bs[k][n]   (contiguous along n: sn == 1; along k (sk == 1): element loads)
// (out of line, like run_jobs: one copy of each variant instead of one per phase keeps the
// kernel's code small enough for the instruction caches)
template <int RPT, int KG, int TRANS>
__device__ __noinline__ void run_tile(const Job& jref, int t, float* smem, const Learn& P, float c1, float c2) {
  TT(0);
  const Job& j = jref;  // in shared memory (run_jobs)
  constexpr int RW = kWarps / KG;  // row-warps
  constexpr int TM = RW * RPT;
  const int ntn = (j.N + kTN - 1) / kTN;
  const int m0 = (t / ntn) * TM, n0 = (t % ntn) * kTN;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kgi = warp % KG, rw = warp / KG, c = lane;
  const int kc_max = (kSmemFloats / (TM + kBS)) & ~3;
  float acc[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) acc[q] = 0.0f;
  const bool b_rows = j.b.sn == 1 && (j.b.sk & 3) == 0 && al16(j.b.p);
  for (int k0 = 0; k0 < j.K; k0 += kc_max) {
    const int kc = min(kc_max, j.K - k0);
    const int kcp = (kc + 3) & ~3;
    float* As = smem;                 // TRANS ? [kcp][TM] : [TM][kcp]
    float* Bs = smem + TM * kcp;      // [kcp][kBS]
    __syncthreads();
    // ---- A
    if (!TRANS) {
      // this warp's row pointers first: gathered rows read their ring index from global
      // memory, so all of them are in flight together instead of one round trip per row
      constexpr int RPW = (TM + kWarps - 1) / kWarps;
      const float* rows[RPW];
#pragma unroll
      for (int q = 0; q < RPW; ++q) {
        const int rr = warp + q * kWarps, m = m0 + rr;
        rows[q] = (rr < TM && m < j.M) ? j.a.row(m) : nullptr;
      }
#pragma unroll
      for (int q = 0; q < RPW; ++q) {
        const int rr = warp + q * kWarps;
        if (rr >= TM) break;
        float* dst = As + rr * kcp;
        if (!rows[q]) {
          for (int kk = lane; kk < kcp; kk += 32) dst[kk] = 0.0f;
          continue;
        }
        const float* src = rows[q] + k0;
        if (al16(src)) {
          const int k4 = kc & ~3;
          for (int kk = 4 * lane; kk < k4; kk += 128) cp_async16(dst + kk, src + kk);
          for (int kk = k4 + lane; kk < kcp; kk += 32) dst[kk] = kk < kc ? __ldcg(src + kk) : 0.0f;
        } else {
          for (int kk = lane; kk < kcp; kk += 32) dst[kk] = kk < kc ? __ldcg(src + kk) : 0.0f;
        }
      }
    } else {
      // source rows of this warp's k steps, one per lane, fetched together (gathered rows read
      // their ring index from global memory) and handed out by shuffles
      const float* lrow = nullptr;
      {
        const int kk = warp + kWarps * lane;
        if (kk < kc) lrow = j.a.row(k0 + kk);
      }
      int it = 0;
      for (int kk = warp; kk < kcp; kk += kThreads / 32, ++it) {
        float* dst = As + kk * TM;
        if (kk >= kc) {
          for (int rr = lane; rr < TM; rr += 32) dst[rr] = 0.0f;
          continue;
        }
        const float* rowp =
            it < 32 ? reinterpret_cast<const float*>(__shfl_sync(
                          0xffffffffu, static_cast<unsigned long long>(reinterpret_cast<uintptr_t>(lrow)), it))
                    : j.a.row(k0 + kk);
        const float* src = rowp + m0;
        const int mdata = j.a.ones_at >= 0 ? j.a.ones_at : j.M;
        if ((TM & 3) == 0 && al16(src) && m0 + TM <= mdata) {
          for (int rr = 4 * lane; rr < TM; rr += 128) cp_async16(dst + rr, src + rr);
        } else {
          for (int rr = lane; rr < TM; rr += 32) {
            const int m = m0 + rr;
            dst[rr] = m < mdata ? __ldcg(src + rr) : (m == j.a.ones_at ? 1.0f : 0.0f);
          }
        }
      }
    }
    // ---- B (rows [kc, kcp) zero: the padded k steps multiply zeros on both sides)
    for (int e = kc * kBS + tid; e < kcp * kBS; e += kThreads) Bs[e] = 0.0f;
    if (b_rows && n0 + kTN <= j.N) {
      for (int e = tid; e < kc * (kTN / 4); e += kThreads) {
        const int kk = e >> 3, n4 = (e & 7) * 4;
        cp_async16(Bs + kk * kBS + n4, j.b.p + (int64_t)(k0 + kk) * j.b.sk + n0 + n4);
      }
    } else {
      // element loads, 8 in flight per thread
      const int total = kc * kTN;
      for (int e0 = tid; e0 < total; e0 += 8 * kThreads) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * kThreads;
          int kk, nn;
          if (j.b.sn == 1) kk = e / kTN, nn = e % kTN;
          else nn = e / kc, kk = e - nn * kc;
          const int n = n0 + nn;
          v[u] = (e < total && n < j.N) ? __ldcg(j.b.p + (int64_t)(k0 + kk) * j.b.sk + (int64_t)n * j.b.sn) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int e = e0 + u * kThreads;
          if (e >= total) break;
          int kk, nn;
          if (j.b.sn == 1) kk = e / kTN, nn = e % kTN;
          else nn = e / kc, kk = e - nn * kc;
          Bs[kk * kBS + nn] = v[u];
        }
      }
    }
    TT(1);
    cp_async_wait_all();
    __syncthreads();
    TT(2);
    // ---- this warp's K segment (multiples of 4)
    const int seg = ((kcp / 4 + KG - 1) / KG) * 4;
    const int klo = kgi * seg, khi = min(kcp, klo + seg);
    const float* bcol = Bs + c;
    if (!TRANS) {
#pragma unroll 2
      for (int kk = klo; kk < khi; kk += 4) {
        const float b0 = bcol[kk * kBS], b1 = bcol[(kk + 1) * kBS], b2 = bcol[(kk + 2) * kBS],
                    b3 = bcol[(kk + 3) * kBS];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
          const float4 a4 = *reinterpret_cast<const float4*>(As + (rw + RW * q) * kcp + kk);
          acc[q] = fmaf(a4.x, b0, acc[q]);
          acc[q] = fmaf(a4.y, b1, acc[q]);
          acc[q] = fmaf(a4.z, b2, acc[q]);
          acc[q] = fmaf(a4.w, b3, acc[q]);
        }
      }
    } else {
#pragma unroll 4
      for (int kk = klo; kk < khi; ++kk) {
        const float bv = bcol[kk * kBS];
        const float* acol = As + kk * TM + rw;
#pragma unroll
        for (int q = 0; q < RPT; ++q) acc[q] = fmaf(acol[RW * q], bv, acc[q]);
      }
    }
  }
  TT(3);
  // ---- partial sums of the K groups, added in group order
  if (KG > 1) {
    __syncthreads();
    float* red = smem;  // [KG][TM][32]
#pragma unroll
    for (int q = 0; q < RPT; ++q) red[(kgi * TM + rw + RW * q) * kTN + c] = acc[q];
    __syncthreads();
    if (kgi != 0) return;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      float v = red[(rw + RW * q) * kTN + c];
      for (int g = 1; g < KG; ++g) v += red[(g * TM + rw + RW * q) * kTN + c];
      acc[q] = v;
    }
  }
  TT(4);
  const int n = n0 + c;
  if (n >= j.N) return;
  const float bias = j.bias ? __ldcg(j.bias + n) : 0.0f;
  // operands of the epilogue loaded up front (one round trip, not one per row)
  float mk[RPT];
  if (j.epi == 2) {
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int m = m0 + rw + RW * q;
      mk[q] = m < j.M ? __ldcg(j.mask + (int64_t)m * j.ldmask + n) : 0.0f;
    }
  }
  if (!j.adam) {
    float* __restrict__ const out = j.c;
    const int64_t ldc = j.ldc;
    const int M = j.M, epi = j.epi;
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int m = m0 + rw + RW * q;
      if (m >= M) break;
      float v = acc[q] + bias;
      if (epi == 1) v = fmaxf(v, 0.0f);
      if (epi == 2 && !(mk[q] > 0.0f)) v = 0.0f;
      out[(int64_t)m * ldc + n] = v;
    }
  } else {  // Adam (agent.py:229-250) on the finished gradient
    // the job's fields in registers first: the stores below go through generic pointers the
    // compiler cannot tell apart from the job in shared memory
    float* __restrict__ const pm = P.m + j.eoff;
    float* __restrict__ const pv = P.v + j.eoff;
    float* __restrict__ const pp = P.p + j.eoff;
    float* __restrict__ const pg = j.c;
    float* __restrict__ const wt = j.wt;
    const int64_t ldc = j.ldc, wt_ld = j.wt_ld;
    const int M = j.M, wt_rows = wt ? j.wt_rows : 0;
    const float b1 = P.b1, b2 = P.b2, lr = P.lr, eps = P.eps;
    float om[RPT], ov[RPT], op[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int m = m0 + rw + RW * q;
      const int64_t e = (int64_t)m * ldc + n;
      om[q] = ov[q] = op[q] = 0.0f;
      if (m < M) om[q] = __ldcg(pm + e), ov[q] = __ldcg(pv + e), op[q] = __ldcg(pp + e);
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int m = m0 + rw + RW * q;
      if (m >= M) break;
      const float v = acc[q] + bias;
      const int64_t e = (int64_t)m * ldc + n;
      pg[e] = v;
      const float mi = b1 * om[q] + (1.0f - b1) * v;
      const float vi = b2 * ov[q] + (1.0f - b2) * v * v;
      pm[e] = mi;
      pv[e] = vi;
      const float pi = op[q] - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
      pp[e] = pi;
      if (m < wt_rows) wt[(int64_t)n * wt_ld + m] = pi;
    }
  }
  TT(5);
}

template <int TRANS>
__device__ __forceinline__ void run_tile_cfg(const Job& j, int t, float* smem, const Learn& P, float c1, float c2) {
  switch (j.rpt * 16 + j.kg) {
    case 1 * 16 + 1: run_tile<1, 1, TRANS>(j, t, smem, P, c1, c2); break;
    case 2 * 16 + 1: run_tile<2, 1, TRANS>(j, t, smem, P, c1, c2); break;
    case 4 * 16 + 1: run_tile<4, 1, TRANS>(j, t, smem, P, c1, c2); break;
    case 8 * 16 + 1: run_tile<8, 1, TRANS>(j, t, smem, P, c1, c2); break;
    case 1 * 16 + 2: run_tile<1, 2, TRANS>(j, t, smem, P, c1, c2); break;
    case 2 * 16 + 2: run_tile<2, 2, TRANS>(j, t, smem, P, c1, c2); break;
    case 4 * 16 + 2: run_tile<4, 2, TRANS>(j, t, smem, P, c1, c2); break;
    case 1 * 16 + 4: run_tile<1, 4, TRANS>(j, t, smem, P, c1, c2); break;
    case 2 * 16 + 4: run_tile<2, 4, TRANS>(j, t, smem, P, c1, c2); break;
    case 4 * 16 + 4: run_tile<4, 4, TRANS>(j, t, smem, P, c1, c2); break;
    case 1 * 16 + 8: run_tile<1, 8, TRANS>(j, t, smem, P, c1, c2); break;
    case 2 * 16 + 8: run_tile<2, 8, TRANS>(j, t, smem, P, c1, c2); break;
    default: run_tile<1, 8, TRANS>(j, t, smem, P, c1, c2); break;
  }
}

// all tiles of up to 3 independent jobs, spread over the grid
__device__ __noinline__ void run_jobs(const Job* pjobs, int nj, float* smem, const Learn& P, float c1 = 1.0f,
                                      float c2 = 1.0f) {
  // the phase's jobs from the kernel parameters into shared memory (the tile loops reread job
  // fields around their asynchronous copies; shared-memory reads are the cheap ones)
  __shared__ Job jobs[3];
  {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(pjobs);
    uint32_t* dst = reinterpret_cast<uint32_t*>(jobs);
    for (int e = threadIdx.x; e < nj * (int)(sizeof(Job) / 4); e += blockDim.x) dst[e] = src[e];
  }
  __syncthreads();
  int total = 0;
  for (int i = 0; i < nj; ++i) total += jobs[i].tiles();
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    int k = t, i = 0;
    while (k >= jobs[i].tiles()) k -= jobs[i].tiles(), ++i;
    if (jobs[i].a.trans)
      run_tile_cfg<1>(jobs[i], k, smem, P, c1, c2);
    else
      run_tile_cfg<0>(jobs[i], k, smem, P, c1, c2);
  }
}

// Tile shapes of one phase: the smallest row count per tile whose tiles fit one wave of a
// reference 148-SM grid, then row-warps x K-groups for that height (K-groups when K is long).
// A fixed reference grid keeps every summation order a function of the problem alone.
__host__ __device__ void plan_tiles(Job* jobs, int nj) {
  constexpr int kRefGrid = 148;
  int lvl = 0;
  for (; lvl < 6; ++lvl) {
    int total = 0;
    for (int i = 0; i < nj; ++i) {
      int tm = 1 << lvl;
      while (tm > 1 && tm / 2 >= jobs[i].M) tm /= 2;
      total += ((jobs[i].M + tm - 1) / tm) * ((jobs[i].N + kTN - 1) / kTN);
    }
    if (total <= kRefGrid) break;
  }
  for (int i = 0; i < nj; ++i) {
    Job& j = jobs[i];
    int tm = 1 << lvl;
    while (tm > 1 && tm / 2 >= j.M) tm /= 2;
    const int K = j.K;
    switch (tm) {
      case 1: j.rpt = 1, j.kg = 8; break;
      case 2: j.rpt = K >= 256 ? 2 : 1, j.kg = K >= 256 ? 8 : 4; break;
      case 4: j.rpt = K >= 256 ? 2 : 1, j.kg = K >= 256 ? 4 : 2; break;
      case 8: j.rpt = K >= 512 ? 4 : (K >= 128 ? 2 : 1), j.kg = K >= 512 ? 4 : (K >= 128 ? 2 : 1); break;
      case 16: j.rpt = K >= 128 ? 4 : 2, j.kg = K >= 128 ? 2 : 1; break;
      case 32: j.rpt = 4, j.kg = 1; break;
      default: j.rpt = 8, j.kg = 1; break;
    }
  }
}

// warp sum of per-lane partials (fixed xor tree: every lane gets the same value)
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// mean of the advantages z[1..A]: lane-strided partial sums, then the xor tree
__device__ __forceinline__ float adv_mean(const float* z, int A) {
  float s = 0.0f;
  for (int j = 1 + (threadIdx.x & 31); j <= A; j += 32) s += __ldcg(z + j);
  return warp_sum(s) / (float)A;
}

// head outputs of R rows (rows hr[r], weights wh[r] / bh[r]) into registers of every lane,
// in head_row's summation order; the loads of 4 k-steps are issued together
template <int A1M, int R, int U = 4>
__device__ __forceinline__ void head_regs_(const float* const* hr, int H, int A1, const float* const* wh,
                                          const float* const* bh, float (*z)[A1M]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < A1M; ++j) z[r][j] = 0.0f;
  for (int k0 = 0; k0 < H; k0 += U * 32) {
    float x[R][U], w[R][U][A1M];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * 32 + lane;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        x[r][u] = k < H ? __ldcg(hr[r] + k) : 0.0f;
#pragma unroll
        for (int j = 0; j < A1M; ++j) w[r][u][j] = (k < H && j < A1) ? __ldcg(wh[r] + (int64_t)k * A1 + j) : 0.0f;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int j = 0; j < A1M; ++j) z[r][j] = fmaf(x[r][u], w[r][u][j], z[r][j]);
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < A1M; ++j) z[r][j] = warp_sum(z[r][j]) + (j < A1 ? __ldcg(bh[r] + j) : 0.0f);
}

// one head row z = h . Wh + bh by one warp (lanes split H), for heads of <= A1M outputs
template <int A1M>
__device__ __forceinline__ void head_row(const float* hr, int H, int A1, const float* wh, const float* bh, float* z) {
  const int lane = threadIdx.x & 31;
  float s[A1M];
#pragma unroll
  for (int j = 0; j < A1M; ++j) s[j] = 0.0f;
  for (int k = lane; k < H; k += 32) {
    const float x = __ldcg(hr + k);
#pragma unroll
    for (int j = 0; j < A1M; ++j)
      if (j < A1) s[j] = fmaf(x, __ldcg(wh + (int64_t)k * A1 + j), s[j]);
  }
#pragma unroll
  for (int j = 0; j < A1M; ++j) s[j] = warp_sum(s[j]);
  if (lane < A1) {
    float v = 0.0f;
#pragma unroll
    for (int j = 0; j < A1M; ++j)
      if (j == lane) v = s[j];
    z[lane] = v + __ldcg(bh + lane);
  }
}

// One row of the small-head step (1 + A <= A1M outputs) with the head outputs kept in
// registers: forward mode writes Q; learn mode runs the double-DQN TD of sample b.
template <int A1M>
__device__ __noinline__ void small_head_row(const Learn& P, int r, int B, const float* HonL, const float* HtgL,
                                            float* dz, float* lrow, float* dhL, bool fwd_only) {
  const int lane = threadIdx.x & 31;
  const int L = P.L, A = P.A, A1 = A + 1, H = P.d[L];
  const float* w_on = P.p + P.w_off[L];
  const float* b_on = P.p + P.b_off[L];
  if (fwd_only) {
    const float* hr[1] = {HonL + (int64_t)r * H};
    const float* wh[1] = {w_on};
    const float* bh[1] = {b_on};
    float z[1][A1M];
    head_regs_<A1M, 1>(hr, H, A1, wh, bh, z);
    float mean = 0.0f;
#pragma unroll
    for (int j = 1; j < A1M; ++j)
      if (j <= A) mean += z[0][j];
    mean /= (float)A;
#pragma unroll
    for (int a = 0; a + 1 < A1M; ++a)
      if (a < A && lane == a) P.q_out[(int64_t)r * A + a] = z[0][0] + z[0][1 + a] - mean;
    return;
  }
  const int b = r;
  const int64_t row = P.idx[b];
  const float rew = P.r_rewards[row];
  const int a = P.r_actions[row];
  const bool done = P.r_done[row] != 0;
  const float w = P.isw[b];
  uint32_t mbits = 0;
#pragma unroll
  for (int j = 0; j + 1 < A1M; ++j)
    if (j < A && P.r_mask[row * A + j]) mbits |= 1u << j;
  bool later = false;
  for (int k = b + 1 + lane; k < B; k += 32) later |= P.idx[k] == row;
  const float* hr[3] = {HonL + (int64_t)b * H, HonL + (int64_t)(B + b) * H, HtgL + (int64_t)b * H};
  const float* wh[3] = {w_on, w_on, P.tp + P.w_off[L]};
  const float* bh[3] = {b_on, b_on, P.tp + P.b_off[L]};
  // the head dgrad's operands (below) for H <= 256, loaded before the head math: they do not
  // depend on it, and issued here their round trip overlaps the head's
  constexpr int DU = 8;
  const bool dh_pre = A1M <= 3 && H <= 32 * DU;
  const float* hc = HonL + (int64_t)(B + b) * H;
  float dwv[DU][A1M], dhv[DU];
  if (dh_pre) {
#pragma unroll
    for (int u = 0; u < DU; ++u) {
      const int n = u * 32 + lane;
      dhv[u] = n < H ? __ldcg(hc + n) : 0.0f;
#pragma unroll
      for (int k = 0; k < A1M; ++k) dwv[u][k] = (n < H && k < A1) ? __ldcg(w_on + (int64_t)n * A1 + k) : 0.0f;
    }
  }
  float z[3][A1M];  // online next, online cur, target next
  head_regs_<A1M, 3>(hr, H, A1, wh, bh, z);
  float mn = 0.0f, mc = 0.0f, mt = 0.0f;
#pragma unroll
  for (int j = 1; j < A1M; ++j)
    if (j <= A) mn += z[0][j], mc += z[1][j], mt += z[2][j];
  mn /= (float)A, mc /= (float)A, mt /= (float)A;
  // masked argmax, first index among equal maxima (agent.py masked_argmax)
  float best = -INFINITY;
  int bj = -1;
  float qa = 0.0f, tn = 0.0f;
#pragma unroll
  for (int j = 0; j + 1 < A1M; ++j) {
    if (j >= A) break;
    const float qv = z[0][0] + z[0][1 + j] - mn;
    if (((mbits >> j) & 1u) && (bj < 0 || qv > best)) best = qv, bj = j;
    if (j == a) qa = z[1][0] + z[1][1 + j] - mc;
  }
  const bool any = bj >= 0;
  const int a_next = any ? bj : 0;
#pragma unroll
  for (int j = 0; j + 1 < A1M; ++j)
    if (j == a_next) tn = z[2][0] + z[2][1 + j] - mt;
  const float d = (done || !any) ? 1.0f : 0.0f;
  const float target = rew + P.gamma * (1.0f - d) * tn;
  const float tdv = qa - target;
  const float ad = fabsf(tdv);
  const float hub = ad <= P.delta ? 0.5f * tdv * tdv : P.delta * (ad - 0.5f * P.delta);
  const float g = w * fminf(fmaxf(tdv, -P.delta), P.delta) / (float)B;
  if (lane <= A) dz[(int64_t)b * A1 + lane] = lane == 0 ? g : ((lane - 1) == a ? g : 0.0f) - g / (float)A;
  // the head's dgrad for this row, dh_L[b] = relu'(H_L(cur)[b]) * (dz[b] Wh^T): K = 1 + A is tiny,
  // so the row's warp does it here (one fma chain per output, k ascending) instead of a phase
  // of its own; Wh is still the pre-update head (its Adam runs in the next phase)
  {
    float dzk[A1M];
#pragma unroll
    for (int k = 0; k < A1M; ++k) dzk[k] = k == 0 ? g : ((k - 1) == a ? g : 0.0f) - g / (float)A;
    float* out = dhL + (int64_t)b * H;
    if (dh_pre) {
#pragma unroll
      for (int u = 0; u < DU; ++u) {
        const int n = u * 32 + lane;
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < A1M; ++k)
          if (k < A1) acc = fmaf(dzk[k], dwv[u][k], acc);
        const float v = acc + 0.0f;
        if (n < H) out[n] = dhv[u] > 0.0f ? v : 0.0f;
      }
    }
    // 8 columns per lane at a time, every load of the block issued before its first use (the
    // stores of one block could alias the next block's loads for the compiler)
    constexpr int U = 8;
    for (int n0 = 0; n0 < (dh_pre ? 0 : H); n0 += 32 * U) {
      float wv[U][A1M], hv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int n = n0 + u * 32 + lane;
        hv[u] = n < H ? __ldcg(hc + n) : 0.0f;
#pragma unroll
        for (int k = 0; k < A1M; ++k) wv[u][k] = (n < H && k < A1) ? __ldcg(w_on + (int64_t)n * A1 + k) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int n = n0 + u * 32 + lane;
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < A1M; ++k)
          if (k < A1) acc = fmaf(dzk[k], wv[u][k], acc);
        const float v = acc + 0.0f;
        if (n < H) out[n] = hv[u] > 0.0f ? v : 0.0f;
      }
    }
  }
  later = __any_sync(0xffffffffu, later);
  if (lane == 0) {
    P.td[b] = tdv;
    lrow[b] = w * hub;
    if (!later) P.r_prio[row] = fabs((double)tdv) + 1e-6;
  }
}

// ---- forward of a few rows (the act of the search loop) --------------------------------
// One row x [1060] through 256-wide layers is ~0.3 MFLOP: the cost is latency.  Every layer's
// K is split over the grid so each CTA reads a few KB of weights: work item (column tile of
// 32, K-chunk) sums its chunk (8 warps split it, fma chains k ascending, warps added in order)
// into a partial row of the workspace; the consumer of the layer's output adds the chunks in
// chunk order, then bias and relu.  The split is planned against a 144-CTA reference grid,
// so every sum's order is a function of the network alone.  The head (<= 8 outputs) runs in
// one warp per row as in the learn step.
constexpr int kSmallRows = 4;

struct Split {
  int nt, ks, kc;  // column tiles, K-chunks, chunk length
};

__host__ __device__ __forceinline__ Split split_of(int K, int N) {
  constexpr int kRefGrid = 144;  // <= the SMs a launch that leaves one free for the sampler has
  Split sp;
  sp.nt = (N + kTN - 1) / kTN;
  int ks = max(1, kRefGrid / sp.nt);
  ks = min(ks, (K + 7) / 8);  // chunks of >= 8
  sp.kc = (K + ks - 1) / ks;
  sp.ks = (K + sp.kc - 1) / sp.kc;
  return sp;
}

// element (r, k) of layer i's input: the state row (i = 0), else relu(sum of layer i-1's
// chunk partials in chunk order + bias)
__device__ __forceinline__ float small_input(const Learn& P, int i, const float* part_prev, int ks_prev, int R, int r,
                                             int k) {
  if (i == 0) return __ldcg(P.x_in + (int64_t)r * P.x_ld + k);
  const int N = P.d[i];
  float v = __ldcg(part_prev + (int64_t)r * N + k);
  for (int q = 1; q < ks_prev; ++q) v += __ldcg(part_prev + ((int64_t)q * R + r) * N + k);
  return fmaxf(v + __ldcg(P.p + P.b_off[i - 1] + k), 0.0f);
}

template <int R>
__device__ __noinline__ void small_forward(const Learn& P, float* smem) {
  const int L = P.L, A1 = P.A + 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* red = smem;  // [kWarps][R][32]
  if (P.act && blockIdx.x == gridDim.x - 1) parity_act_rows(P.pl);  // ordered before the decision by the barriers
  const float* part_prev = nullptr;
  int ks_prev = 0;
  int64_t off = 0;
  for (int i = 0; i < L; ++i) {
    const int K = P.d[i], N = P.d[i + 1];
    const Split sp = split_of(K, N);
    float* part = P.ws + off;  // [ks][R][N]
    const float* W = P.p + P.w_off[i];
    for (int item = blockIdx.x; item < sp.nt * sp.ks; item += gridDim.x) {
      const int ct = item % sp.nt, kq = item / sp.nt;
      const int n = ct * kTN + lane;
      const int k0 = kq * sp.kc, k1 = min(K, k0 + sp.kc);
      const int kw = (k1 - k0 + kWarps - 1) / kWarps;
      const int wk0 = min(k1, k0 + warp * kw), wk1 = min(k1, wk0 + kw);
      float acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = 0.0f;
      for (int kb = wk0; kb < wk1; kb += 32) {
        const int cnt = min(32, wk1 - kb);
        float x[R];
#pragma unroll
        for (int r = 0; r < R; ++r) x[r] = lane < cnt ? small_input(P, i, part_prev, ks_prev, R, r, kb + lane) : 0.0f;
        float w[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) w[u] = (u < cnt && n < N) ? __ldcg(W + (int64_t)(kb + u) * N + n) : 0.0f;
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          if (u >= cnt) break;
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r] = fmaf(__shfl_sync(0xffffffffu, x[r], u), w[u], acc[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) red[(warp * R + r) * kTN + lane] = acc[r];
      __syncthreads();
      if (warp == 0 && n < N) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float v = red[r * kTN + lane];
          for (int w2 = 1; w2 < kWarps; ++w2) v += red[(w2 * R + r) * kTN + lane];
          part[((int64_t)kq * R + r) * N + n] = v;
        }
      }
      __syncthreads();
    }
    grid_sync(P.bar + 2 + P.reserve);  // one counter word per grid size
    part_prev = part;
    ks_prev = sp.ks;
    off += (int64_t)sp.ks * R * N;
  }
  if (blockIdx.x != 0) return;
  // the last hidden layer's rows, then the head and Q (one warp per row)
  const int H = P.d[L];
  float* hl = P.ws + off;  // [R][H]
  for (int e = tid; e < R * H; e += kThreads) hl[e] = small_input(P, L, part_prev, ks_prev, R, e / H, e % H);
  __syncthreads();
  if (warp < R) {
    if (A1 <= 3)
      small_head_row<3>(P, warp, R, hl, nullptr, nullptr, nullptr, nullptr, true);
    else
      small_head_row<8>(P, warp, R, hl, nullptr, nullptr, nullptr, nullptr, true);
  }
  if (!P.act) return;
  __syncthreads();
  if (tid == 0) {
    parity_step_begin(P.pl, false, true);  // active; slot / size before the push
    parity_act_decide(P.pl, P.q_out, P.action);
  }
}

__host__ __device__ __forceinline__ AOp rows_of(const float* p, int64_t sr) {
  return AOp{p, sr, nullptr, nullptr, nullptr, 0, 0, -1};
}

// Every phase's jobs and the workspace carve-up, planned once on the host (they depend on the
// network, the batch and the buffers only) and read by the kernel from its parameters: no
// per-phase setup on the critical path.  Phase order: the L forward layers, the wide head's
// forward (heads of > 7 actions), the head backward (wide heads), the L backward layers.
void plan_phases(Learn& P) {
  const int L = P.L, A1 = P.A + 1;
  const bool fwd_only = P.rows_fwd > 0;
  const int B = fwd_only ? P.rows_fwd : P.B;
  const int Ron = fwd_only ? B : 2 * B;  // online rows: [next; cur]
  // workspace: online activations [Ron, d_i], target activations [B, d_i] (i = 1..L),
  // head outputs, dz, dh_i [B, d_i], the per-row loss terms
  float* ws = P.ws;
  for (int i = 1; i <= L; ++i) {
    P.Hon[i] = ws;
    ws += (int64_t)Ron * P.d[i];
    P.Htg[i] = ws;
    ws += (int64_t)B * P.d[i];
    P.dh[i] = ws;
    ws += (int64_t)B * P.d[i];
  }
  P.zon = ws;
  ws += (int64_t)Ron * A1;
  P.ztg = ws;
  ws += (int64_t)B * A1;
  P.dz = ws;
  ws += (int64_t)B * A1;
  P.lrow = ws;
  P.nph = 0;
  // forward, layer by layer
  for (int i = 0; i < L; ++i) {
    Phase& ph = P.ph[P.nph++];
    const int K = P.d[i], N = P.d[i + 1];
    ph.nj = 0;
    Job& on = ph.jobs[ph.nj++];
    on = Job{};
    if (i == 0)
      on.a = fwd_only ? rows_of(P.x_in, P.x_ld) : AOp{nullptr, P.r_ld, P.r_next, P.r_states, P.idx, B, 0, -1};
    else
      on.a = rows_of(P.Hon[i], P.d[i]);
    on.b = BOp{P.p + P.w_off[i], N, 1};
    on.c = P.Hon[i + 1];
    on.ldc = N;
    on.M = Ron, on.N = N, on.K = K;
    on.bias = P.p + P.b_off[i];
    on.epi = 1;
    if (!fwd_only) {
      Job& tg = ph.jobs[ph.nj++];
      tg = on;
      tg.a = i == 0 ? AOp{nullptr, P.r_ld, P.r_next, P.r_next, P.idx, B, 0, -1} : rows_of(P.Htg[i], P.d[i]);
      tg.b = BOp{P.tp + P.w_off[i], N, 1};
      tg.c = P.Htg[i + 1];
      tg.M = B;
      tg.bias = P.tp + P.b_off[i];
    }
    plan_tiles(ph.jobs, ph.nj);
  }
  const int H = P.d[L];
  const bool small_head = A1 <= 8;
  if (!small_head) {  // head outputs as tiles over the grid
    Phase& ph = P.ph[P.nph++];
    ph.nj = 0;
    Job& on = ph.jobs[ph.nj++];
    on = Job{};
    on.a = rows_of(P.Hon[L], H);
    on.b = BOp{P.p + P.w_off[L], A1, 1};
    on.c = P.zon;
    on.ldc = A1;
    on.M = Ron, on.N = A1, on.K = H;
    on.bias = P.p + P.b_off[L];
    if (!fwd_only) {
      Job& tg = ph.jobs[ph.nj++];
      tg = on;
      tg.a = rows_of(P.Htg[L], H);
      tg.b = BOp{P.tp + P.w_off[L], A1, 1};
      tg.c = P.ztg;
      tg.M = B;
      tg.bias = P.tp + P.b_off[L];
    }
    plan_tiles(ph.jobs, ph.nj);
  }
  if (fwd_only) return;
  // Each weight-gradient tile sums the whole batch, so it applies Adam itself; a weight's
  // transposed copy is refreshed one phase later when a dgrad of its own phase reads it.
  auto with_adam = [&](Job& j, int s, bool direct_wt) {
    j.adam = 1;
    j.eoff = P.w_off[s];
    j.wt = direct_wt ? P.wt[s] : nullptr;
    j.wt_ld = P.wt_ld[s];
    j.wt_rows = P.d[s];
  };
  const float* Hc = P.Hon[L] + (int64_t)B * H;  // current-state rows of the last hidden layer
  if (!small_head) {
    // head backward: gWh = H_L(cur)^T dz, gbh, dh_L = relu'(H_L) * (dz Wh^T); Adam on Wh, bh.
    // (Small heads: dh_L comes with the TD rows and gWh joins the next phase.)
    Phase& ph = P.ph[P.nph++];
    ph.nj = 2;
    Job& wg = ph.jobs[0];
    wg = Job{};
    // (m=j, k=b) = Hc[b][j]; row H of ones: the bias gradient lands right after gWh (bh follows wh)
    wg.a = AOp{Hc, H, nullptr, nullptr, nullptr, 0, 1, H};
    wg.b = BOp{P.dz, A1, 1};
    wg.c = P.grad + P.w_off[L];
    wg.ldc = A1;
    wg.M = H + 1, wg.N = A1, wg.K = B;
    with_adam(wg, L, false);
    Job& dg = ph.jobs[1];
    dg = Job{};
    dg.a = rows_of(P.dz, A1);
    // (k=a, n=j) = Wh[j][a]: rows of the transposed copy (the pre-update weights)
    dg.b = BOp{P.wt[L], P.wt_ld[L], 1};
    dg.c = P.dh[L];
    dg.ldc = H;
    dg.M = B, dg.N = H, dg.K = A1;
    dg.epi = 2;
    dg.mask = Hc;
    dg.ldmask = H;
    plan_tiles(ph.jobs, 2);
  }
  // hidden layers, last to first: gW_{i-1} (+ Adam), dh_{i-1}
  for (int i = L; i >= 1; --i) {
    Phase& ph = P.ph[P.nph++];
    const int din = P.d[i - 1], dout = P.d[i];
    ph.nj = 0;
    Job& wg = ph.jobs[ph.nj++];
    wg = Job{};
    // (m=p, k=b) = input row b, column p; row din of ones gives gb right after gW (b_i follows w_i)
    if (i == 1)
      wg.a = AOp{nullptr, P.r_ld, P.r_states, P.r_states, P.idx, B, 1, din};
    else
      wg.a = AOp{P.Hon[i - 1] + (int64_t)B * din, din, nullptr, nullptr, nullptr, 0, 1, din};
    wg.b = BOp{P.dh[i], dout, 1};
    wg.c = P.grad + P.w_off[i - 1];
    wg.ldc = dout;
    wg.M = din + 1, wg.N = dout, wg.K = B;
    with_adam(wg, i - 1, i == 1 && !P.lazy_wt0);  // no dgrad reads w_0's copy: written directly (or left)
    if (i > 1) {
      Job& dg = ph.jobs[ph.nj++];
      dg = Job{};
      dg.a = rows_of(P.dh[i], dout);
      // (k=q, n=p) = W[p][q] = row q of the transposed copy (pre-update)
      dg.b = BOp{P.wt[i - 1], P.wt_ld[i - 1], 1};
      dg.c = P.dh[i - 1];
      dg.ldc = din;
      dg.M = B, dg.N = din, dg.K = dout;
      dg.epi = 2;
      dg.mask = P.Hon[i - 1] + (int64_t)B * din;
      dg.ldmask = din;
    }
    if (i == L && small_head) {
      // gWh = H_L(cur)^T dz + Adam; no job of this phase reads the head's transposed copy, so
      // the epilogue writes it directly
      Job& hg = ph.jobs[ph.nj++];
      hg = Job{};
      hg.a = AOp{Hc, H, nullptr, nullptr, nullptr, 0, 1, H};
      hg.b = BOp{P.dz, A1, 1};
      hg.c = P.grad + P.w_off[L];
      hg.ldc = A1;
      hg.M = H + 1, hg.N = A1, hg.K = B;
      with_adam(hg, L, true);
    }
    plan_tiles(ph.jobs, ph.nj);
  }
}

__global__ void __launch_bounds__(kThreads, 1) mlp_fused_kernel(const __grid_constant__ Learn P) {
  extern __shared__ float smem[];
  // every CTA alike (no barrier is entered): the self-gated loop body's learn waits for a full
  // batch in the ring and stops with the loop (act of the step saw the budget spent)
  if (P.gate > 0 && (P.ctl[AP_CTL_SIZE] < P.gate || !P.ctl[AP_PL_ACTIVE])) return;
  if (P.act) {
    // every CTA decides alike from words nobody writes during the act; CTA 0 records it
    // after the first grid barrier (all reads are done by then)
    const bool active = parity_step_begin(P.pl, true, false);
    if (!active) {
      if (blockIdx.x == 0 && threadIdx.x == 0) P.pl.ctl[AP_PL_ACTIVE] = 0;
      return;
    }
    // an exploring step needs no Q (agent.py:166-168: the random() draw decides first), so every
    // CTA replays that draw and, when it explores, only CTA 0 stays to take the step's action
    uint64_t w6[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) w6[k] = P.pl.rng[k];
    NpPcg64 g = NpPcg64::load(w6);
    if (g.next_double() < epsilon_at(P.pl.ctl[AP_CTL_TRAIN], P.pl.eps_start, P.pl.eps_final, P.pl.eps_decay)) {
      if (blockIdx.x != 0) return;
      parity_act_rows(P.pl);
      __syncthreads();
      if (threadIdx.x == 0) {
        parity_step_begin(P.pl, false, true);
        parity_act_decide(P.pl, P.q_out, P.action);
      }
      return;
    }
  }
  // this learn step's train counter, read by every CTA before the first grid barrier (CTA 0
  // advances it at the end, in parity-tail mode)
  const int64_t t_train = P.ctl ? P.ctl[AP_CTL_TRAIN] : 0;
  if (P.rng_from && blockIdx.x == 0 && threadIdx.x < 6) P.rng_to[threadIdx.x] = P.rng_from[threadIdx.x];
  int tk = 0;
#ifdef AP_FUSED_TILE_TRACE
  if (blockIdx.x == 0 && threadIdx.x == 0) g_tile_trace = P.trace, g_tile_n = 0;
#endif
  trace_mark(P.trace, tk);
  const int L = P.L, A = P.A, A1 = A + 1;
  const bool fwd_only = P.rows_fwd > 0;
  const int B = fwd_only ? P.rows_fwd : P.B;
  const int Ron = fwd_only ? B : 2 * B;  // online rows: [next; cur]
  const bool t0 = threadIdx.x == 0;
  if (fwd_only && B <= kSmallRows && A1 <= 8) {
    switch (B) {
      case 1: small_forward<1>(P, smem); break;
      case 2: small_forward<2>(P, smem); break;
      case 3: small_forward<3>(P, smem); break;
      default: small_forward<4>(P, smem); break;
    }
    return;
  }
  int ph = 0;
  // forward, layer by layer
  for (int i = 0; i < L; ++i, ++ph) {
    run_jobs(P.ph[ph].jobs, P.ph[ph].nj, smem, P);
    trace_arrive(P.trace, tk);
    grid_sync(P.bar);
    trace_mark(P.trace, tk);
  }
  // head outputs: wide heads as tiles over the grid (then a barrier), small heads inside the
  // per-row step below (one warp computes its row's 1 or 3 head rows itself)
  const int H = P.d[L];
  const bool small_head = A1 <= 8;
  if (!small_head) {
    run_jobs(P.ph[ph].jobs, P.ph[ph].nj, smem, P);
    ++ph;
    trace_arrive(P.trace, tk);
    grid_sync(P.bar);
    trace_mark(P.trace, tk);
  }
  {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5), nw = gridDim.x * kWarps;
    float* const zon = P.zon;
    float* const ztg = P.ztg;
    float* const dz = P.dz;
    const float* const HonL = P.Hon[L];
    const float* const HtgL = P.Htg[L];
    for (int r = gw; r < (fwd_only ? Ron : B); r += nw) {
      if (small_head) {
        if (A1 <= 3)
          small_head_row<3>(P, r, B, HonL, HtgL, dz, P.lrow, P.dh[L], fwd_only);
        else
          small_head_row<8>(P, r, B, HonL, HtgL, dz, P.lrow, P.dh[L], fwd_only);
        continue;
      }
      if (fwd_only) {
        if (small_head) {
          head_row<8>(HonL + (int64_t)r * H, H, A1, P.p + P.w_off[L], P.p + P.b_off[L], zon + (int64_t)r * A1);
          __syncwarp();
        }
        // Q = V + A - mean(A) (agent.py dueling head)
        const float* z = zon + (int64_t)r * A1;
        const float mean = adv_mean(z, A), v0 = __ldcg(z);
        for (int a2 = lane; a2 < A; a2 += 32) P.q_out[(int64_t)r * A + a2] = v0 + __ldcg(z + 1 + a2) - mean;
        continue;
      }
      // double-DQN TD (agent.py:277-296) for row b = r: online next -> best action over the next
      // mask, target next -> its value, online cur -> Q of the taken action
      const int b = r;
      const int64_t row = P.idx[b];
      // the row's replay fields, loaded before the head math they do not depend on
      const float rew = P.r_rewards[row];
      const int a = P.r_actions[row];
      const bool done = P.r_done[row] != 0;
      const float w = P.isw[b];
      const uint8_t* mk = P.r_mask + row * A;
      bool later = false;
      for (int k = b + 1 + lane; k < B; k += 32) later |= P.idx[k] == row;
      if (small_head) {
        head_row<8>(HonL + (int64_t)b * H, H, A1, P.p + P.w_off[L], P.p + P.b_off[L], zon + (int64_t)b * A1);
        head_row<8>(HonL + (int64_t)(B + b) * H, H, A1, P.p + P.w_off[L], P.p + P.b_off[L],
                    zon + (int64_t)(B + b) * A1);
        head_row<8>(HtgL + (int64_t)b * H, H, A1, P.tp + P.w_off[L], P.tp + P.b_off[L], ztg + (int64_t)b * A1);
        __syncwarp();
      }
      const float* zn = zon + (int64_t)b * A1;
      const float* zt = ztg + (int64_t)b * A1;
      const float* zc = zon + (int64_t)(B + b) * A1;
      const float mn = adv_mean(zn, A), mt = adv_mean(zt, A), mc = adv_mean(zc, A);
      // masked argmax, the first index among equal maxima (lane-strided, then a tie-aware tree)
      float best = -INFINITY;
      int bj = -1;
      const float zn0 = __ldcg(zn);
      for (int j2 = lane; j2 < A; j2 += 32) {
        if (!mk[j2]) continue;
        const float qv = zn0 + __ldcg(zn + 1 + j2) - mn;
        if (bj < 0 || qv > best) best = qv, bj = j2;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (oj >= 0 && (bj < 0 || ob > best || (ob == best && oj < bj))) best = ob, bj = oj;
      }
      const bool any = bj >= 0;
      const int a_next = any ? bj : 0;
      const float d = (done || !any) ? 1.0f : 0.0f;
      const float target = rew + P.gamma * (1.0f - d) * (__ldcg(zt) + __ldcg(zt + 1 + a_next) - mt);
      const float tdv = (__ldcg(zc) + __ldcg(zc + 1 + a) - mc) - target;
      const float ad = fabsf(tdv);
      const float hub = ad <= P.delta ? 0.5f * tdv * tdv : P.delta * (ad - 0.5f * P.delta);
      const float g = w * fminf(fmaxf(tdv, -P.delta), P.delta) / (float)B;
      for (int j2 = lane; j2 <= A; j2 += 32)
        dz[(int64_t)b * A1 + j2] = j2 == 0 ? g : ((j2 - 1) == a ? g : 0.0f) - g / (float)A;
      // priorities[idx] = |td| + 1e-6; among duplicate indices the last write wins (agent.py:226)
      later = __any_sync(0xffffffffu, later);
      if (lane == 0) {
        P.td[b] = tdv;
        P.lrow[b] = w * hub;
        if (!later) P.r_prio[row] = fabs((double)tdv) + 1e-6;
      }
    }
  }
  if (fwd_only) return;
  trace_arrive(P.trace, tk);
  grid_sync(P.bar);
  trace_mark(P.trace, tk);
  if (P.pstat && blockIdx.x == gridDim.x - 1) {
    // the ring's max priority after this step's updates (the next push writes it; agent.py:199)
    // and the cached powers of the updated priorities, by the last CTA, which the following
    // phases load least (duplicate indices write the same final value)
    for (int b = threadIdx.x; b < B; b += kThreads) {
      const int64_t row = P.idx[b];
      P.r_scaled[row] = pow(__ldcg(P.r_prio + row), P.alpha);
    }
    const int64_t size = P.ctl[AP_CTL_SIZE];
    float* red = smem + kSmemFloats - 512;
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < size; i += kThreads) m = fmax(m, __ldcg(P.r_prio + i));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    double* dred = reinterpret_cast<double*>(red);
    if ((threadIdx.x & 31) == 0) dred[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int k = 1; k < kWarps; ++k) m = fmax(m, dred[k]);
      m = fmax(m, dred[0]);
      P.pstat[0] = size ? m : 1.0;
      P.pstat[1] = pow(P.pstat[0], P.alpha);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // fixed-order sum; the terms loaded in parallel
    float* sl = smem + kSmemFloats - 256;       // (past every tile's footprint in this phase)
    for (int b = threadIdx.x; b < B; b += 32) sl[b] = __ldcg(P.lrow + b);
    __syncwarp();
    if (threadIdx.x == 0) {
      float s = 0.0f;
      for (int b = 0; b < B; ++b) s += sl[b];
      *P.loss = s;
    }
  }

  // Adam bias corrections (host values, or the parity loop's table entry for this train step)
  float c1 = P.c1, c2 = P.c2;
  if (P.ctab) {
    const int64_t k = t_train + P.t_offset - P.ctl[AP_PL_TAB_BASE];
    c1 = P.ctab[2 * k];
    c2 = P.ctab[2 * k + 1];
  }
  auto refresh_wt = [&](int s) {
    const int rows = P.d[s], cols = P.d[s + 1];
    const float* w = P.p + P.w_off[s];
    float* dst = P.wt[s];
    const int64_t ld = P.wt_ld[s];
    for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < (int64_t)rows * cols;
         e += (int64_t)gridDim.x * kThreads) {
      const int64_t c = e / rows, r = e - c * rows;
      dst[c * ld + r] = __ldcg(w + r * cols + c);
    }
  };

  if (!small_head) {
    run_jobs(P.ph[ph].jobs, P.ph[ph].nj, smem, P, c1, c2);
    ++ph;
    trace_arrive(P.trace, tk);
    grid_sync(P.bar);
    trace_mark(P.trace, tk);
  }
  // hidden layers, last to first: gW_{i-1} (+ Adam), dh_{i-1}; refresh the transposed copy of
  // the weight updated in the phase before
  for (int i = L; i >= 1; --i, ++ph) {
    run_jobs(P.ph[ph].jobs, P.ph[ph].nj, smem, P, c1, c2);
    if (i < L || !small_head) refresh_wt(i);  // i == L: the head; else w_i (updated in the phase of layer i + 1)
    if (i > 1) {
      trace_arrive(P.trace, tk);
      grid_sync(P.bar);
      trace_mark(P.trace, tk);
    }
  }
  trace_arrive(P.trace, tk);
  trace_mark(P.trace, tk);
  if (!P.tail_ctl) return;
  // parity-loop tail (agent.py:325-337): every CTA read the train counter before the first
  // barrier, so CTA 0 may advance it now
  if (blockIdx.x == 0 && t0) {
    const int64_t k = t_train - P.tail_ctl[AP_PL_TRAIN0];
    const float v = *P.loss;
    if (k >= 0 && k < P.loss_cap) P.loss_log[k] = v;
    if (!isfinite(v) && P.tail_ctl[AP_PL_LOSS_BAD] < 0) P.tail_ctl[AP_PL_LOSS_BAD] = k;
    P.tail_ctl[AP_CTL_TRAIN] = t_train + 1;
  }
  if ((t_train + 1) % P.sync_every != 0) return;
  // hard target sync: online parameters and transposed copies -> the target's, once every
  // CTA's Adam updates and copy refreshes are done
  grid_sync(P.bar);
  for (int k = 0; k < P.sync_n; ++k) {
    const float4* src = reinterpret_cast<const float4*>(P.sync_src[k]);
    float4* dst = reinterpret_cast<float4*>(P.sync_dst[k]);
    const int64_t n4 = P.sync_count[k] / 4;
    for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < n4; e += (int64_t)gridDim.x * kThreads)
      dst[e] = __ldcg(src + e);
    for (int64_t e = 4 * n4 + (int64_t)blockIdx.x * kThreads + threadIdx.x; e < P.sync_count[k];
         e += (int64_t)gridDim.x * kThreads)
      P.sync_dst[k][e] = __ldcg(P.sync_src[k] + e);
  }
}

int64_t workspace_floats(int L, const int* d, int B, bool fwd_only) {
  const int64_t Ron = fwd_only ? B : 2 * B;
  int64_t n = 0;
  for (int i = 1; i <= L; ++i) n += (Ron + 2 * (int64_t)B) * d[i];
  const int64_t A1 = d[L + 1];
  n += (Ron + 2 * (int64_t)B) * A1 + B + 64;
  if (fwd_only && B <= kSmallRows && A1 <= 8) {  // small_forward: chunk partials + the last hidden rows
    int64_t s = (int64_t)B * d[L];
    for (int i = 0; i < L; ++i) s += (int64_t)split_of(d[i], d[i + 1]).ks * B * d[i + 1];
    n = std::max(n, s);
  }
  return n;
}

int launch(const Learn& P, cudaStream_t stream, int reserve_sms = 0) {
  int sms = 0;
  if (int rc = current_sm_count(&sms)) return rc;
  sms = std::max(1, sms - reserve_sms);
  static PerDeviceMax configured;
  const int smem = kSmemFloats * 4 + 64;
  if (configured.need(current_device(), smem))
    AP_CUDA_CHECK(cudaFuncSetAttribute(mlp_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(kThreads);
  // the few-row forward (small_forward) needs only its warp-reduction buffer
  const bool small = P.rows_fwd > 0 && P.rows_fwd <= kSmallRows && P.A + 1 <= 8;
  cfg.dynamicSmemBytes = small ? kWarps * kSmallRows * kTN * 4 : smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the grid barriers cannot deadlock
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  AP_CUDA_CHECK(cudaLaunchKernelEx(&cfg, mlp_fused_kernel, P));
  return AP_OK;
}

bool fill_net(Learn* P, int32_t L, const int32_t* dims, const int64_t* w_off, const int64_t* b_off) {
  if (L < 1 || L > kMaxLayers) return false;
  P->L = L;
  for (int i = 0; i <= L + 1; ++i) {
    P->d[i] = dims[i];
    if (dims[i] < 1) return false;
  }
  P->A = dims[L + 1] - 1;
  for (int i = 0; i <= L; ++i) P->w_off[i] = w_off[i], P->b_off[i] = b_off[i];
  return P->A >= 1;
}

}  // namespace
}  // namespace apb

using namespace apb;

extern "C" {

int64_t ap_mlp_fused_workspace(int32_t L, const int32_t* dims, int32_t rows, int32_t forward_only) {
  if (L < 1 || L > kMaxLayers || !dims || rows < 1) return -1;
  return workspace_floats(L, dims, rows, forward_only != 0);
}

int ap_mlp_forward_fused(int32_t L, const int32_t* dims, const int64_t* w_off, const int64_t* b_off,
                         const float* params, const float* x, int64_t ldx, int32_t rows, float* q, float* workspace,
                         uint32_t* barrier, void* stream) {
  Learn P = {};
  if (!fill_net(&P, L, dims, w_off, b_off) || !params || !x || !q || !workspace || !barrier || rows < 1 ||
      rows > 256) {
    set_error("ap_mlp_forward_fused: bad arguments (1..4 hidden layers, 1..256 rows)");
    return AP_ERR_INVALID;
  }
  P.rows_fwd = rows;
  P.p = const_cast<float*>(params);
  P.tp = params;
  P.x_in = x;
  P.x_ld = ldx;
  P.q_out = q;
  P.ws = workspace;
  P.bar = barrier;
  plan_phases(P);
  return launch(P, (cudaStream_t)stream);
}

int ap_parity_act_fused(const ap_parity_loop* pl, int32_t L, const int32_t* dims, const int64_t* w_off,
                        const int64_t* b_off, const float* params, float* q, float* workspace, uint32_t* barrier,
                        int32_t* action, void* stream) {
  Learn P = {};
  if (!pl || !pl->ctl || !pl->rng || !pl->state || !fill_net(&P, L, dims, w_off, b_off) || !params || !q ||
      !workspace || !barrier || !action || P.A + 1 > 8 || P.A != pl->num_actions) {
    set_error("ap_parity_act_fused: bad arguments (1..4 hidden layers, 1 <= A <= 7 actions matching the loop)");
    return AP_ERR_INVALID;
  }
  P.rows_fwd = 1;
  P.p = const_cast<float*>(params);
  P.tp = params;
  P.x_in = pl->state;
  P.x_ld = dims[0];
  P.q_out = q;
  P.ws = workspace;
  P.bar = barrier;
  P.act = 1;
  P.pl = *pl;
  P.action = action;
  // early PER sample: one SM stays free for the sampler the act's decision waits for
  P.reserve = pl->early_sample ? 1 : 0;
  return launch(P, (cudaStream_t)stream, P.reserve);
}

int ap_dqn_learn_fused(const ap_fused_learn* a, void* stream) {
  Learn P = {};
  if (!a || !fill_net(&P, a->L, a->dims, a->w_off, a->b_off) || a->batch < 1 || a->batch > 256 || !a->params ||
      !a->target || !a->idx || !a->weights || !a->grad || !a->m || !a->v || !a->workspace || !a->barrier) {
    set_error("ap_dqn_learn_fused: bad arguments");
    return AP_ERR_INVALID;
  }
  for (int i = 0; i <= a->L; ++i)
    if (!a->wt[i] || a->wt_ld[i] < a->dims[i]) {
      set_error("ap_dqn_learn_fused: every weight needs its transposed copy (wt[i], wt_ld[i] >= dims[i])");
      return AP_ERR_INVALID;
    }
  P.B = a->batch;
  P.p = a->params;
  P.tp = a->target;
  P.r_states = a->r_states;
  P.r_next = a->r_next;
  P.r_ld = a->r_ld;
  P.r_actions = a->r_actions;
  P.r_rewards = a->r_rewards;
  P.r_done = a->r_done;
  P.r_mask = a->r_mask;
  P.r_prio = a->r_prio;
  P.idx = a->idx;
  P.isw = a->weights;
  P.gamma = a->gamma;
  P.delta = a->huber_delta;
  P.grad = a->grad;
  P.m = a->m;
  P.v = a->v;
  P.nparams = a->nparams;
  P.lr = a->lr;
  P.b1 = a->beta1;
  P.b2 = a->beta2;
  P.eps = a->eps;
  P.c1 = a->correct1;
  P.c2 = a->correct2;
  P.ctab = a->ctab;
  P.ctl = a->ctl;
  P.t_offset = a->t_offset;
  for (int i = 0; i <= a->L; ++i) {
    P.wt[i] = a->wt[i];
    P.wt_ld[i] = a->wt_ld[i];
  }
  P.td = a->td;
  P.loss = a->loss;
  P.ws = a->workspace;
  P.bar = a->barrier;
  P.trace = reinterpret_cast<unsigned long long*>(a->trace);
  P.gate = a->ctl ? a->gate : 0;
  if (a->tail_ctl) {
    if (!a->ctl || a->tail_ctl != a->ctl || !a->loss_log || a->sync_every < 1 || a->sync_n < 0 || a->sync_n > 6) {
      set_error("ap_dqn_learn_fused: the tail needs ctl == tail_ctl, loss_log, sync_every >= 1, <= 6 sync segments");
      return AP_ERR_INVALID;
    }
    for (int k = 0; k < a->sync_n; ++k)
      if (!a->sync_src[k] || !a->sync_dst[k] || a->sync_count[k] < 0 || (reinterpret_cast<uintptr_t>(a->sync_src[k]) & 15) ||
          (reinterpret_cast<uintptr_t>(a->sync_dst[k]) & 15)) {
        set_error("ap_dqn_learn_fused: sync segments need 16-byte aligned non-null pointers");
        return AP_ERR_INVALID;
      }
    P.tail_ctl = a->tail_ctl;
    P.loss_log = a->loss_log;
    P.loss_cap = a->loss_cap;
    P.sync_every = a->sync_every;
    P.sync_n = a->sync_n;
    for (int k = 0; k < a->sync_n; ++k)
      P.sync_src[k] = a->sync_src[k], P.sync_dst[k] = a->sync_dst[k], P.sync_count[k] = a->sync_count[k];
    if (a->rng_from && a->rng_to) P.rng_from = a->rng_from, P.rng_to = a->rng_to;
  }
  P.r_scaled = a->r_scaled;
  if (a->r_scaled && !a->pstat) {
    set_error("ap_dqn_learn_fused: the priority-power cache needs pstat");
    return AP_ERR_INVALID;
  }
  P.pstat = a->r_scaled ? a->pstat : nullptr;
  P.alpha = a->per_alpha;
  P.lazy_wt0 = a->lazy_wt0;
  plan_phases(P);
  return launch(P, (cudaStream_t)stream);
}

}  // extern "C"
