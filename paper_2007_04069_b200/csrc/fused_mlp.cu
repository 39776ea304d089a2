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
constexpr int kMaxLayers = 4;  // hidden layers
constexpr int kTN = 32;        // tile columns (one per lane)
constexpr int kSmemFloats = 50 * 1024;  // 200 KB of dynamic shared memory per CTA

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
};

// grid-wide barrier (all CTAs co-resident: cooperative launch); generation counter in bar[1]
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned gen;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(bar + 1) : "memory");
      } while (cur == gen);
    }
    __threadfence();
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
// relu' mask from `mask` rows (2), none (0).  Tiles of 8 * rpt rows x 32 columns.
struct Job {
  AOp a;
  BOp b;
  float* c;
  int64_t ldc;
  int M, N, K, rpt;
  const float* bias;
  int epi;
  const float* mask;
  int64_t ldmask;
  __device__ __forceinline__ int tiles() const { return ((M + 8 * rpt - 1) / (8 * rpt)) * ((N + kTN - 1) / kTN); }
};

template <int RPT>
__device__ void run_tile(const Job& j, int t, float* smem) {
  const int tm_rows = 8 * RPT;
  const int ntn = (j.N + kTN - 1) / kTN;
  const int m0 = (t / ntn) * tm_rows, n0 = (t % ntn) * kTN;
  const int tid = threadIdx.x, r = tid >> 5, c = tid & 31;
  // chunk of K that fits: As [tm_rows][kc] + Bs [kc][33]
  const int kc_max = kSmemFloats / (tm_rows + kTN + 1);
  float acc[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) acc[q] = 0.0f;
  for (int k0 = 0; k0 < j.K; k0 += kc_max) {
    const int kc = min(kc_max, j.K - k0);
    float* As = smem;                  // [tm_rows][kc]
    float* Bs = smem + tm_rows * kc;   // [kc][33]
    __syncthreads();
    if (!j.a.trans) {
      for (int e = tid; e < tm_rows * kc; e += kThreads) {
        const int rr = e / kc, kk = e - rr * kc;
        const int m = m0 + rr;
        As[e] = m < j.M ? __ldcg(j.a.row(m) + k0 + kk) : 0.0f;
      }
    } else {
      for (int e = tid; e < tm_rows * kc; e += kThreads) {
        const int kk = e / tm_rows, rr = e - kk * tm_rows;
        const int m = m0 + rr;
        As[rr * kc + kk] = m < j.M ? __ldcg(j.a.row(k0 + kk) + m) : 0.0f;
      }
    }
    for (int e = tid; e < kc * kTN; e += kThreads) {
      int kk, nn;
      if (j.b.sn == 1) {
        kk = e / kTN, nn = e - kk * kTN;
      } else {
        nn = e / kc, kk = e - nn * kc;
      }
      const int n = n0 + nn;
      Bs[kk * (kTN + 1) + nn] = n < j.N ? __ldcg(j.b.p + (int64_t)(k0 + kk) * j.b.sk + (int64_t)n * j.b.sn) : 0.0f;
    }
    __syncthreads();
    const float* bcol = Bs + c;
    for (int kk = 0; kk < kc; ++kk) {
      const float bv = bcol[kk * (kTN + 1)];
#pragma unroll
      for (int q = 0; q < RPT; ++q) acc[q] = fmaf(As[(r + 8 * q) * kc + kk], bv, acc[q]);
    }
  }
  const int n = n0 + c;
  if (n >= j.N) return;
  const float bias = j.bias ? __ldcg(j.bias + n) : 0.0f;
#pragma unroll
  for (int q = 0; q < RPT; ++q) {
    const int m = m0 + r + 8 * q;
    if (m >= j.M) break;
    float v = acc[q] + bias;
    if (j.epi == 1) v = fmaxf(v, 0.0f);
    if (j.epi == 2 && !(__ldcg(j.mask + (int64_t)m * j.ldmask + n) > 0.0f)) v = 0.0f;
    j.c[(int64_t)m * j.ldc + n] = v;
  }
}

// all tiles of up to 3 independent jobs, spread over the grid
__device__ void run_jobs(const Job* jobs, int nj, float* smem) {
  int total = 0;
  for (int i = 0; i < nj; ++i) total += jobs[i].tiles();
  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    int k = t, i = 0;
    while (k >= jobs[i].tiles()) k -= jobs[i].tiles(), ++i;
    switch (jobs[i].rpt) {
      case 1: run_tile<1>(jobs[i], k, smem); break;
      case 2: run_tile<2>(jobs[i], k, smem); break;
      case 4: run_tile<4>(jobs[i], k, smem); break;
      default: run_tile<8>(jobs[i], k, smem); break;
    }
  }
}

// column sums out[n] = sum_{m < M} x[m * ld + n] (bias gradients), rows in order
__device__ void colsum(const float* x, int64_t ld, int M, int N, float* out) {
  for (int n = blockIdx.x * kThreads + threadIdx.x; n < N; n += gridDim.x * kThreads) {
    float s = 0.0f;
    for (int m = 0; m < M; ++m) s += __ldcg(x + (int64_t)m * ld + n);
    out[n] = s;
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
        on.a = AOp{P.x_in, P.x_ld, nullptr, nullptr, nullptr, 0, 0};
      } else {
        on.a = AOp{nullptr, P.r_ld, P.r_next, P.r_states, P.idx, B, 0};
      }
    } else {
      on.a = AOp{Hon[i], P.d[i], nullptr, nullptr, nullptr, 0, 0};
    }
    on.b = BOp{P.p + P.w_off[i], N, 1};
    on.c = Hon[i + 1];
    on.ldc = N;
    on.M = Ron, on.N = N, on.K = K;
    on.rpt = Ron >= 64 ? 2 : 1;
    on.bias = P.p + P.b_off[i];
    on.epi = 1;
    if (!fwd_only) {
      Job& tg = jobs[nj++];
      tg = on;
      tg.a = i == 0 ? AOp{nullptr, P.r_ld, P.r_next, P.r_next, P.idx, B, 0} : AOp{Htg[i], P.d[i], nullptr, nullptr,
                                                                                    nullptr, 0, 0};
      tg.b = BOp{P.tp + P.w_off[i], N, 1};
      tg.c = Htg[i + 1];
      tg.M = B;
      tg.rpt = 1;
      tg.bias = P.tp + P.b_off[i];
    }
    run_jobs(jobs, nj, smem);
    grid_sync(P.bar);
  }

  // head + dueling (+ TD, loss, priorities): one CTA
  const int H = P.d[L];
  if (blockIdx.x == 0) {
    const float* wh = P.p + P.w_off[L];
    const float* bh = P.p + P.b_off[L];
    const float* twh = P.tp + P.w_off[L];
    const float* tbh = P.tp + P.b_off[L];
    const int nrows = fwd_only ? Ron : Ron + B;
    for (int e = threadIdx.x; e < nrows * A1; e += kThreads) {
      const int row = e / A1, j = e - row * A1;
      const bool tgt = row >= Ron;
      const float* h = tgt ? Htg[L] + (int64_t)(row - Ron) * H : Hon[L] + (int64_t)row * H;
      const float* w = tgt ? twh : wh;
      float s = 0.0f;
      for (int k = 0; k < H; ++k) s = fmaf(__ldcg(h + k), __ldcg(w + (int64_t)k * A1 + j), s);
      s += __ldcg((tgt ? tbh : bh) + j);
      (tgt ? ztg + (int64_t)(row - Ron) * A1 : zon + (int64_t)row * A1)[j] = s;
    }
    __syncthreads();
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
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int b = 0; b < B; ++b) s += lrow[b];
        *P.loss = s;
        for (int b = 0; b < B; ++b) P.r_prio[P.idx[b]] = fabs((double)P.td[b]) + 1e-6;  // last duplicate wins
      }
    }
  }
  if (fwd_only) return;
  grid_sync(P.bar);

  // head backward: gWh = H_L(cur)^T dz, gbh, dh_L = relu'(H_L) * (dz Wh^T)
  {
    const float* Hc = Hon[L] + (int64_t)B * H;  // current-state rows
    Job jobs[2];
    jobs[0] = Job{};
    jobs[0].a = AOp{Hc, H, nullptr, nullptr, nullptr, 0, 1};  // (m=j, k=b) = Hc[b][j]
    jobs[0].b = BOp{dz, A1, 1};
    jobs[0].c = P.grad + P.w_off[L];
    jobs[0].ldc = A1;
    jobs[0].M = H, jobs[0].N = A1, jobs[0].K = B, jobs[0].rpt = 4;
    jobs[1] = Job{};
    jobs[1].a = AOp{dz, A1, nullptr, nullptr, nullptr, 0, 0};
    jobs[1].b = BOp{P.p + P.w_off[L], 1, A1};  // (k=a, n=j) = Wh[j][a]
    jobs[1].c = dh[L];
    jobs[1].ldc = H;
    jobs[1].M = B, jobs[1].N = H, jobs[1].K = A1, jobs[1].rpt = 1;
    jobs[1].epi = 2;
    jobs[1].mask = Hc;
    jobs[1].ldmask = H;
    run_jobs(jobs, 2, smem);
    colsum(dz, A1, B, A1, P.grad + P.b_off[L]);
  }
  grid_sync(P.bar);

  // hidden layers, last to first
  for (int i = L; i >= 1; --i) {
    const int din = P.d[i - 1], dout = P.d[i];
    Job jobs[2];
    int nj = 0;
    Job& wg = jobs[nj++];
    wg = Job{};
    if (i == 1)
      wg.a = AOp{nullptr, P.r_ld, P.r_states, P.r_states, P.idx, B, 1};  // (m=p, k=b) = state row idx[b], col p
    else
      wg.a = AOp{Hon[i - 1] + (int64_t)B * din, din, nullptr, nullptr, nullptr, 0, 1};
    wg.b = BOp{dh[i], dout, 1};
    wg.c = P.grad + P.w_off[i - 1];
    wg.ldc = dout;
    wg.M = din, wg.N = dout, wg.K = B, wg.rpt = 8;
    if (i > 1) {
      Job& dg = jobs[nj++];
      dg = Job{};
      dg.a = AOp{dh[i], dout, nullptr, nullptr, nullptr, 0, 0};
      dg.b = BOp{P.p + P.w_off[i - 1], 1, dout};  // (k=q, n=p) = W[p][q]
      dg.c = dh[i - 1];
      dg.ldc = din;
      dg.M = B, dg.N = din, dg.K = dout, dg.rpt = 1;
      dg.epi = 2;
      dg.mask = Hon[i - 1] + (int64_t)B * din;
      dg.ldmask = din;
    }
    run_jobs(jobs, nj, smem);
    colsum(dh[i], dout, B, dout, P.grad + P.b_off[i - 1]);
    grid_sync(P.bar);
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
  return launch(P, (cudaStream_t)stream);
}

}  // extern "C"
