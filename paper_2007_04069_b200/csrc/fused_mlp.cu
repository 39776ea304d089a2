// Fused dueling-MLP learner and forward for small batches (the parity agent and
// the device search loop): one persistent kernel per DQN learn step.
//
// The reference learner (agent.py:258-299) at its batch of 64 is three small
// forwards (online and target on the next states, online on the states), a
// double-DQN TD with Huber and importance weights, the analytic backward of a
// dueling MLP and Adam.  As separate tensor-core GEMMs that is ~40 dependent
// launches of 4-11 us each; here every phase is a set of register-tiled fp32
// tiles spread over all SMs, with grid-wide barriers between dependent phases
// (2L + 3 for L hidden layers), so one launch does the whole step:
//
//   fwd layer i   H_i = relu(H_{i-1} W_i + b_i)   online rows [next; cur], target rows next
//                 (layer 0 reads the replay-ring rows through the sampled indices)
//   head + TD     z = H_L Wh + bh, Q = V + A - mean(A), double-DQN target, Huber,
//                 dz = dLoss/dz, td, loss, priorities |td| + 1e-6 (last duplicate wins)
//   head bwd      gWh = H_L^T dz, gbh = colsum dz, dh_L = relu'(H_L) (dz Wh^T)
//   layer i bwd   gW_i = H_{i-1}^T dh_i, gb_i = colsum dh_i, dh_{i-1} = relu'(H_{i-1}) (dh_i W_i^T)
//   Adam          every parameter, plus the transposed weight copies the tensor-core
//                 forward path reads
//
// Every sum runs in a fixed order (k ascending inside a tile, tiles never split K),
// so results are deterministic and independent of the grid size.  fp32 products
// and sums (FMA) track the fp64 reference to ~1e-6 relative (tests/test_fused_mlp_gpu.py).
// The same kernel in forward mode gives Q for a few rows (the act of the search loop).
#include <algorithm>
#include <cstdint>

#include "engine.h"

namespace apb {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxLayers = 4;  // hidden layers
constexpr int kTN = 32;        // tile columns (one per lane)
constexpr int kSmemFloats = 56 * 1024;  // 224 KB of dynamic shared memory per CTA (one chunk at K <= 1100)

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
};

__device__ __forceinline__ void trace_mark(unsigned long long* tr, int& k) {
  if (tr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    tr[k] = t;
  }
  ++k;
}

// grid-wide barrier (all CTAs co-resident: cooperative launch).  bar[0] counts arrivals
// monotonically (it stays a multiple of the grid size between launches): one release add per
// CTA, then acquire loads until the count reaches the next multiple.  The CTA barrier before
// the add orders every thread's writes before thread 0's release (cumulativity).
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned old;
    asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
    const unsigned target = (old / gridDim.x + 1) * gridDim.x;
    unsigned cur;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar) : "memory");
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
  __device__ __forceinline__ const float* row(int r) const {
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
  __device__ __forceinline__ int tm() const { return (kWarps / kg) * rpt; }
  __device__ __forceinline__ int tiles() const { return ((M + tm() - 1) / tm()) * ((N + kTN - 1) / kTN); }
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
template <int RPT, int KG, int TRANS>
__device__ void run_tile(const Job& j, int t, float* smem) {
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
      for (int rr = warp; rr < TM; rr += kThreads / 32) {
        const int m = m0 + rr;
        float* dst = As + rr * kcp;
        if (m >= j.M) {
          for (int kk = lane; kk < kcp; kk += 32) dst[kk] = 0.0f;
          continue;
        }
        const float* src = j.a.row(m) + k0;
        if (al16(src)) {
          const int k4 = kc & ~3;
          for (int kk = 4 * lane; kk < k4; kk += 128) cp_async16(dst + kk, src + kk);
          for (int kk = k4 + lane; kk < kcp; kk += 32) dst[kk] = kk < kc ? __ldcg(src + kk) : 0.0f;
        } else {
          for (int kk = lane; kk < kcp; kk += 32) dst[kk] = kk < kc ? __ldcg(src + kk) : 0.0f;
        }
      }
    } else {
      for (int kk = warp; kk < kcp; kk += kThreads / 32) {
        float* dst = As + kk * TM;
        if (kk >= kc) {
          for (int rr = lane; rr < TM; rr += 32) dst[rr] = 0.0f;
          continue;
        }
        const float* src = j.a.row(k0 + kk) + m0;
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
    cp_async_wait_all();
    __syncthreads();
    // ---- this warp's K segment (multiples of 4)
    const int seg = ((kcp / 4 + KG - 1) / KG) * 4;
    const int klo = kgi * seg, khi = min(kcp, klo + seg);
    const float* bcol = Bs + c;
    if (!TRANS) {
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
  const int n = n0 + c;
  if (n >= j.N) return;
  const float bias = j.bias ? __ldcg(j.bias + n) : 0.0f;
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int m = m0 + rw + RW * q;
    if (m >= j.M) break;
    float v = acc[q] + bias;
    if (j.epi == 1) v = fmaxf(v, 0.0f);
    if (j.epi == 2 && !(__ldcg(j.mask + (int64_t)m * j.ldmask + n) > 0.0f)) v = 0.0f;
    j.c[(int64_t)m * j.ldc + n] = v;
  }
}

template <int TRANS>
__device__ __forceinline__ void run_tile_cfg(const Job& j, int t, float* smem) {
  switch (j.rpt * 16 + j.kg) {
    case 1 * 16 + 1: run_tile<1, 1, TRANS>(j, t, smem); break;
    case 2 * 16 + 1: run_tile<2, 1, TRANS>(j, t, smem); break;
    case 4 * 16 + 1: run_tile<4, 1, TRANS>(j, t, smem); break;
    case 8 * 16 + 1: run_tile<8, 1, TRANS>(j, t, smem); break;
    case 1 * 16 + 2: run_tile<1, 2, TRANS>(j, t, smem); break;
    case 2 * 16 + 2: run_tile<2, 2, TRANS>(j, t, smem); break;
    case 4 * 16 + 2: run_tile<4, 2, TRANS>(j, t, smem); break;
    case 1 * 16 + 4: run_tile<1, 4, TRANS>(j, t, smem); break;
    case 2 * 16 + 4: run_tile<2, 4, TRANS>(j, t, smem); break;
    case 4 * 16 + 4: run_tile<4, 4, TRANS>(j, t, smem); break;
    case 1 * 16 + 8: run_tile<1, 8, TRANS>(j, t, smem); break;
    case 2 * 16 + 8: run_tile<2, 8, TRANS>(j, t, smem); break;
    default: run_tile<1, 8, TRANS>(j, t, smem); break;
  }
}

// all tiles of up to 3 independent jobs, spread over the grid
__device__ void run_jobs(const Job* jobs, int nj, float* smem) {
  int total = 0;
  for (int i = 0; i < nj; ++i) total += jobs[i].tiles();
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    int k = t, i = 0;
    while (k >= jobs[i].tiles()) k -= jobs[i].tiles(), ++i;
    if (jobs[i].a.trans)
      run_tile_cfg<1>(jobs[i], k, smem);
    else
      run_tile_cfg<0>(jobs[i], k, smem);
  }
}

// head outputs z[row] = h[row] . Wh + bh for many rows: one warp per row, lanes split H
template <int A1M>
__device__ void head_rows(const float* h, int64_t ldh, int rows, int H, int A1, const float* wh, const float* bh,
                          float* z, int wbase, int wstride) {
  const int lane = threadIdx.x & 31;
  for (int row = wbase; row < rows; row += wstride) {
    float s[A1M];
#pragma unroll
    for (int j = 0; j < A1M; ++j) s[j] = 0.0f;
    const float* hr = h + (int64_t)row * ldh;
    for (int k = lane; k < H; k += 32) {
      const float x = __ldcg(hr + k);
#pragma unroll
      for (int j = 0; j < A1M; ++j)
        if (j < A1) s[j] = fmaf(x, __ldcg(wh + (int64_t)k * A1 + j), s[j]);
    }
#pragma unroll
    for (int j = 0; j < A1M; ++j)
      for (int o = 16; o; o >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
    if (lane < A1) {
      float v = 0.0f;
#pragma unroll
      for (int j = 0; j < A1M; ++j)
        if (j == lane) v = s[j];
      z[(int64_t)row * A1 + lane] = v + __ldcg(bh + lane);
    }
  }
}

__device__ __forceinline__ float dueling_q(const float* z, int A, int a) {
  float mean = 0.0f;
  for (int j = 1; j <= A; ++j) mean += z[j];
  mean /= (float)A;
  return z[0] + z[1 + a] - mean;
}

__global__ void __launch_bounds__(kThreads, 1) mlp_fused_kernel(Learn P) {
  extern __shared__ float smem[];
  int tk = 0;
  trace_mark(P.trace, tk);
  const int L = P.L, A = P.A, A1 = A + 1;
  const bool fwd_only = P.rows_fwd > 0;
  const int B = fwd_only ? P.rows_fwd : P.B;
  const int Ron = fwd_only ? B : 2 * B;  // online rows: [next; cur]
  // workspace: online activations [Ron, d_i], target activations [B, d_i] (i = 1..L),
  // head outputs, dz, dh_i [B, d_i]
  float* ws = P.ws;
  float* Hon[kMaxLayers + 1];
  float* Htg[kMaxLayers + 1];
  float* dh[kMaxLayers + 1];
  for (int i = 1; i <= L; ++i) {
    Hon[i] = ws;
    ws += (int64_t)Ron * P.d[i];
    Htg[i] = ws;
    ws += (int64_t)B * P.d[i];
    dh[i] = ws;
    ws += (int64_t)B * P.d[i];
  }
  float* zon = ws;
  ws += (int64_t)Ron * A1;
  float* ztg = ws;
  ws += (int64_t)B * A1;
  float* dz = ws;
  ws += (int64_t)B * A1;

  // forward, layer by layer
  for (int i = 0; i < L; ++i) {
    const int K = P.d[i], N = P.d[i + 1];
    Job jobs[2];
    int nj = 0;
    Job& on = jobs[nj++];
    on = Job{};
    if (i == 0) {
      if (fwd_only) {
        on.a = AOp{P.x_in, P.x_ld, nullptr, nullptr, nullptr, 0, 0, -1};
      } else {
        on.a = AOp{nullptr, P.r_ld, P.r_next, P.r_states, P.idx, B, 0, -1};
      }
    } else {
      on.a = AOp{Hon[i], P.d[i], nullptr, nullptr, nullptr, 0, 0, -1};
    }
    on.b = BOp{P.p + P.w_off[i], N, 1};
    on.c = Hon[i + 1];
    on.ldc = N;
    on.M = Ron, on.N = N, on.K = K;
    // small row counts split K over the warps (the act forward: 1 row), large ones split rows
    on.rpt = Ron >= 64 ? 2 : 1;
    on.kg = Ron >= 64 ? 2 : (Ron >= 8 ? 4 : 8);
    on.bias = P.p + P.b_off[i];
    on.epi = 1;
    if (!fwd_only) {
      Job& tg = jobs[nj++];
      tg = on;
      tg.a = i == 0 ? AOp{nullptr, P.r_ld, P.r_next, P.r_next, P.idx, B, 0, -1} : AOp{Htg[i], P.d[i], nullptr, nullptr,
                                                                                    nullptr, 0, 0, -1};
      tg.b = BOp{P.tp + P.w_off[i], N, 1};
      tg.c = Htg[i + 1];
      tg.M = B;
      tg.rpt = 2;
      tg.kg = 2;
      tg.bias = P.tp + P.b_off[i];
    }
    run_jobs(jobs, nj, smem);
    grid_sync(P.bar);
    trace_mark(P.trace, tk);
  }

  // head outputs, one warp per row over the whole grid (online rows, then target rows)
  const int H = P.d[L];
  {
    const int wid = blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5), nw = gridDim.x * (kThreads / 32);
    if (A1 <= 8) {
      head_rows<8>(Hon[L], H, Ron, H, A1, P.p + P.w_off[L], P.p + P.b_off[L], zon, wid, nw);
      if (!fwd_only) head_rows<8>(Htg[L], H, B, H, A1, P.tp + P.w_off[L], P.tp + P.b_off[L], ztg, wid, nw);
    } else {
      // wide heads: one thread per (row, output)
      const int tid = blockIdx.x * kThreads + threadIdx.x, nt = gridDim.x * kThreads;
      const int nrows = fwd_only ? Ron : Ron + B;
      for (int e = tid; e < nrows * A1; e += nt) {
        const int row = e / A1, jj = e - row * A1;
        const bool tgt = row >= Ron;
        const float* h = tgt ? Htg[L] + (int64_t)(row - Ron) * H : Hon[L] + (int64_t)row * H;
        const float* w = (tgt ? P.tp : P.p) + P.w_off[L];
        float acc = 0.0f;
        for (int k = 0; k < H; ++k) acc = fmaf(__ldcg(h + k), __ldcg(w + (int64_t)k * A1 + jj), acc);
        acc += __ldcg((tgt ? P.tp : P.p) + P.b_off[L] + jj);
        (tgt ? ztg + (int64_t)(row - Ron) * A1 : zon + (int64_t)row * A1)[jj] = acc;
      }
    }
  }
  grid_sync(P.bar);
    trace_mark(P.trace, tk);
  if (blockIdx.x == 0) {
    if (fwd_only) {
      for (int e = threadIdx.x; e < Ron * A; e += kThreads) {
        const int row = e / A, a = e - row * A;
        P.q_out[(int64_t)row * A + a] = dueling_q(zon + (int64_t)row * A1, A, a);
      }
    } else {
      // double-DQN TD (agent.py:277-296) for row b: online next -> best action over the next mask,
      // target next -> its value, online cur -> Q of the taken action
      float* lrow = smem;  // [B] weighted Huber terms
      for (int b = threadIdx.x; b < B; b += kThreads) {
        const int64_t row = P.idx[b];
        const uint8_t* mk = P.r_mask + row * A;
        const float* zn = zon + (int64_t)b * A1;
        bool any = false;
        float best = -INFINITY;
        int best_j = 0;
        for (int j = 0; j < A; ++j) {
          if (!mk[j]) continue;
          const float qv = dueling_q(zn, A, j);
          if (!any || qv > best) best = qv, best_j = j;
          any = true;
        }
        const int a_next = any ? best_j : 0;
        const float d = (P.r_done[row] || !any) ? 1.0f : 0.0f;
        const float target =
            P.r_rewards[row] + P.gamma * (1.0f - d) * dueling_q(ztg + (int64_t)b * A1, A, a_next);
        const int a = P.r_actions[row];
        const float tdv = dueling_q(zon + (int64_t)(B + b) * A1, A, a) - target;
        const float w = P.isw[b];
        const float ad = fabsf(tdv);
        const float hub = ad <= P.delta ? 0.5f * tdv * tdv : P.delta * (ad - 0.5f * P.delta);
        const float g = w * fminf(fmaxf(tdv, -P.delta), P.delta) / (float)B;
        for (int j = 0; j <= A; ++j) dz[(int64_t)b * A1 + j] = j == 0 ? g : ((j - 1) == a ? g : 0.0f) - g / (float)A;
        P.td[b] = tdv;
        lrow[b] = w * hub;
        // priorities[idx] = |td| + 1e-6; among duplicate indices the last write wins (agent.py:226)
        bool last = true;
        for (int k = b + 1; k < B; ++k) last &= P.idx[k] != row;
        if (last) P.r_prio[row] = fabs((double)tdv) + 1e-6;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int b = 0; b < B; ++b) s += lrow[b];
        *P.loss = s;
      }
    }
  }
  if (fwd_only) return;
  grid_sync(P.bar);
    trace_mark(P.trace, tk);

  // head backward: gWh = H_L(cur)^T dz, gbh, dh_L = relu'(H_L) * (dz Wh^T)
  {
    const float* Hc = Hon[L] + (int64_t)B * H;  // current-state rows
    Job jobs[2];
    jobs[0] = Job{};
    // (m=j, k=b) = Hc[b][j]; row H of ones: the bias gradient lands right after gWh (bh follows wh)
    jobs[0].a = AOp{Hc, H, nullptr, nullptr, nullptr, 0, 1, H};
    jobs[0].b = BOp{dz, A1, 1};
    jobs[0].c = P.grad + P.w_off[L];
    jobs[0].ldc = A1;
    jobs[0].M = H + 1, jobs[0].N = A1, jobs[0].K = B, jobs[0].rpt = 4, jobs[0].kg = 1;
    jobs[1] = Job{};
    jobs[1].a = AOp{dz, A1, nullptr, nullptr, nullptr, 0, 0, -1};
    // (k=a, n=j) = Wh[j][a]: rows of the transposed copy when present (16-byte staging)
    jobs[1].b = P.wt[L] ? BOp{P.wt[L], P.wt_ld[L], 1} : BOp{P.p + P.w_off[L], 1, A1};
    jobs[1].c = dh[L];
    jobs[1].ldc = H;
    jobs[1].M = B, jobs[1].N = H, jobs[1].K = A1, jobs[1].rpt = 1, jobs[1].kg = 1;
    jobs[1].epi = 2;
    jobs[1].mask = Hc;
    jobs[1].ldmask = H;
    run_jobs(jobs, 2, smem);
  }
  grid_sync(P.bar);
    trace_mark(P.trace, tk);

  // hidden layers, last to first
  for (int i = L; i >= 1; --i) {
    const int din = P.d[i - 1], dout = P.d[i];
    Job jobs[2];
    int nj = 0;
    Job& wg = jobs[nj++];
    wg = Job{};
    // (m=p, k=b) = input row b, column p; row din of ones gives gb right after gW (b_i follows w_i)
    if (i == 1)
      wg.a = AOp{nullptr, P.r_ld, P.r_states, P.r_states, P.idx, B, 1, din};
    else
      wg.a = AOp{Hon[i - 1] + (int64_t)B * din, din, nullptr, nullptr, nullptr, 0, 1, din};
    wg.b = BOp{dh[i], dout, 1};
    wg.c = P.grad + P.w_off[i - 1];
    wg.ldc = dout;
    wg.M = din + 1, wg.N = dout, wg.K = B, wg.rpt = 4, wg.kg = 1;
    if (i > 1) {
      Job& dg = jobs[nj++];
      dg = Job{};
      dg.a = AOp{dh[i], dout, nullptr, nullptr, nullptr, 0, 0, -1};
      // (k=q, n=p) = W[p][q] = row q of the transposed copy
      dg.b = P.wt[i - 1] ? BOp{P.wt[i - 1], P.wt_ld[i - 1], 1} : BOp{P.p + P.w_off[i - 1], 1, dout};
      dg.c = dh[i - 1];
      dg.ldc = din;
      dg.M = B, dg.N = din, dg.K = dout, dg.rpt = 1, dg.kg = 2;
      dg.epi = 2;
      dg.mask = Hon[i - 1] + (int64_t)B * din;
      dg.ldmask = din;
    }
    run_jobs(jobs, nj, smem);
    grid_sync(P.bar);
    trace_mark(P.trace, tk);
  }

  // Adam (agent.py:229-250) over every parameter + the transposed weight copies
  float c1 = P.c1, c2 = P.c2;
  if (P.ctab) {
    const int64_t k = P.ctl[AP_CTL_TRAIN] + P.t_offset - P.ctl[AP_PL_TAB_BASE];
    c1 = P.ctab[2 * k];
    c2 = P.ctab[2 * k + 1];
  }
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < P.nparams; e += (int64_t)gridDim.x * kThreads) {
    const float gi = __ldcg(P.grad + e);
    const float mi = P.b1 * P.m[e] + (1.0f - P.b1) * gi;
    const float vi = P.b2 * P.v[e] + (1.0f - P.b2) * gi * gi;
    P.m[e] = mi;
    P.v[e] = vi;
    const float pi = P.p[e] - P.lr * (mi / c1) / (sqrtf(vi / c2) + P.eps);
    P.p[e] = pi;
    for (int s = 0; s <= L; ++s) {
      const int64_t off = P.w_off[s], rows = P.d[s], cols = P.d[s + 1];
      if (e >= off && e < off + rows * cols && P.wt[s]) {
        const int64_t rr = (e - off) / cols, cc = (e - off) - rr * cols;
        P.wt[s][cc * P.wt_ld[s] + rr] = pi;
      }
    }
  }
  trace_mark(P.trace, tk);
}

int64_t workspace_floats(int L, const int* d, int B, bool fwd_only) {
  const int64_t Ron = fwd_only ? B : 2 * B;
  int64_t n = 0;
  for (int i = 1; i <= L; ++i) n += (Ron + 2 * (int64_t)B) * d[i];
  const int64_t A1 = d[L + 1];
  return n + (Ron + 2 * (int64_t)B) * A1 + 64;
}

int launch(const Learn& P, cudaStream_t stream) {
  int sms = 0;
  if (int rc = current_sm_count(&sms)) return rc;
  static PerDeviceMax configured;
  const int smem = kSmemFloats * 4 + 64;
  if (configured.need(current_device(), smem))
    AP_CUDA_CHECK(cudaFuncSetAttribute(mlp_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
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
  return launch(P, (cudaStream_t)stream);
}

int ap_dqn_learn_fused(const ap_fused_learn* a, void* stream) {
  Learn P = {};
  if (!a || !fill_net(&P, a->L, a->dims, a->w_off, a->b_off) || a->batch < 1 || a->batch > 256 || !a->params ||
      !a->target || !a->idx || !a->weights || !a->grad || !a->m || !a->v || !a->workspace || !a->barrier) {
    set_error("ap_dqn_learn_fused: bad arguments");
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
  return launch(P, (cudaStream_t)stream);
}

}  // extern "C"
