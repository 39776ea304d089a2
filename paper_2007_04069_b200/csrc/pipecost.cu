// K2 / K3 — pipeline cost model on the device, bit-exact with the reference.
//
// Reference: pipecost.py:72-336 (stage_metrics, pipeline_length,
// memory_feasible, proportional_device_counts/cuts, candidate_pivots),
// topology.py:121-148 (transfer / ring allreduce), envs.py:371-404
// (PipeTrainEnv._state), envs.py:593-616 (PipeInferEnv decode + length).
//
// Bit parity rules (SURVEY §7 hard part 1), all enforced here:
//  * this file is compiled with -fmad=false: every + and * rounds on its own;
//  * stage compute sums are naive sequential sums starting at each stage's
//    first instruction (never prefix differences);
//  * CPython >= 3.12 builtin sum() over floats is Neumaier-compensated
//    (py_sum below), e.g. pipeline_length's sum(times) and the total of
//    proportional_device_counts;
//  * byte counts are integers (exact in int64, converted once);
//  * expressions keep Python's left-to-right association, ties in max/min
//    and in the largest-remainder sort resolve to the lowest index.
//
// K2 layout: a candidate list bound with ap_pipe_train_table gets a table of
// every stage sum its plans can have (each entry summed in the reference's
// order), so ap_pipe_train_state / ap_pipe_metrics_bound read stage sums
// instead of re-summing the cost array (train_state_tab_kernel, one CTA per
// env, features + block normalisation + one-hot fused).  Unbound lists take
// the per-env-reuse sweep (train_prefix_kernel + train_tail_kernel) or, with
// AP_PP_FULL=1, one sequential sweep per candidate (train_cand_kernel).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "engine.h"

namespace apb {
namespace {

constexpr int kMaxStages = 32;

struct Topo {
  int32_t g;  // gpus per server
  int32_t d;  // devices
  double intra, inter;
};

__host__ __device__ inline double bw(const Topo& t, int a, int b) { return (a / t.g == b / t.g) ? t.intra : t.inter; }

// CPython 3.12 builtin sum() of floats (Python/bltinmodule.c, Neumaier)
__host__ __device__ inline double py_sum(const double* x, int n) {
  if (n <= 0) return 0.0;
  double total = x[0];
  double c = 0.0;
  for (int i = 1; i < n; ++i) {
    const double v = x[i];
    const double t = total + v;
    if (fabs(total) >= fabs(v))
      c += (total - t) + v;
    else
      c += (v - t) + total;
    total = t;
  }
  if (c != 0.0 && isfinite(c)) total += c;
  return total;
}

// proportional_device_counts (pipecost.py:207-237)
__host__ __device__ inline void proportional_counts(const double* comp, int k, int d, int* counts) {
  const double total = py_sum(comp, k);
  double q[kMaxStages];
  int sum = 0;
  for (int i = 0; i < k; ++i) {
    q[i] = total <= 0.0 ? (double)d / (double)k : ((double)d * comp[i]) / total;
    counts[i] = (int)(long long)q[i];
    sum += counts[i];
  }
  const int rem = d - sum;
  int add[kMaxStages];
  for (int i = 0; i < k; ++i) {
    const double fi = q[i] - (double)counts[i];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double fj = q[j] - (double)counts[j];
      rank += (fj > fi) || (fj == fi && j < i);
    }
    add[i] = rank < rem;
  }
  for (int i = 0; i < k; ++i) counts[i] += add[i];
  for (;;) {  // starvation fix: no stage keeps zero devices
    int poorest = -1;
    for (int i = 0; i < k; ++i)
      if (counts[i] == 0) {
        poorest = i;
        break;
      }
    if (poorest < 0) break;
    int richest = 0;
    for (int i = 1; i < k; ++i)
      if (counts[i] > counts[richest]) richest = i;
    counts[richest] -= 1;
    counts[poorest] = 1;
  }
}

// ring allreduce over devices [start, end) (topology.py:131-148)
__host__ __device__ inline double allreduce(const Topo& t, double bytes, int start, int end,
                                            const double* fac = nullptr) {
  const int n = end - start;
  if (n <= 1 || bytes == 0.0) return 0.0;
  // the slowest link of the ring start -> .. -> end-1 -> start, in closed form
  // (the reference walks the n links): one server -> all intra; otherwise the
  // wrap link is inter-server, the n-1 consecutive links cross `hops` server
  // boundaries, and the rest are intra.  min() over the same link set.
  const int s0 = start / t.g, s1 = (end - 1) / t.g;
  const bool has_inter = s0 != s1, has_intra = s0 == s1 || n - 1 > s1 - s0;
  double slow = INFINITY;
  if (has_inter && t.inter < slow) slow = t.inter;
  if (has_intra && t.intra < slow) slow = t.intra;
  // fac (optional): fac[n] = (2.0 * (n - 1)) / n precomputed with the same operations
  return (fac ? fac[n] : (2.0 * (double)(n - 1)) / (double)n) * bytes / slow;
}

// transfer between consecutive groups (topology.py:121-128)
__host__ __device__ inline double transfer(const Topo& t, double bytes, int src, int dst) {
  if (src == dst) return 0.0;
  return bytes / bw(t, src, dst);
}

__host__ __device__ inline void groups_from_counts(const int* counts, int k, int* start, int* end) {
  int acc = 0;
  for (int s = 0; s < k; ++s) {
    start[s] = acc;
    acc += counts[s];
    end[s] = acc;
  }
}

// builtin sum() over numpy float64 scalars: not PyFloat_CheckExact, so CPython
// takes its generic PyNumber_Add path — a plain left-to-right sum
__host__ __device__ inline double naive_sum(const double* x, int n) {
  double total = 0.0;
  for (int i = 0; i < n; ++i) total = (i == 0) ? x[0] : total + x[i];
  return total;
}

// pipeline_length (pipecost.py:144-176) for groups [start, end).  `exact_floats`
// selects CPython's compensated float sum (metrics are Python floats, as from
// stage_metrics) or the naive generic sum (numpy scalars, as from
// PipeInferEnv.decode_metrics, envs.py:608-615).
__host__ __device__ inline double pipeline_len(const Topo& t, int k, int m, const double* comp, const double* act,
                                               const double* param, const int* start, const int* end,
                                               bool exact_floats = true) {
  double times[kMaxStages], trans[kMaxStages], red_max = 0.0, t_max = 0.0;
  for (int s = 0; s < k; ++s) {
    times[s] = (comp[s] / 1000.0) / (double)(end[s] - start[s]);
    if (s == 0 || times[s] > t_max) t_max = times[s];
    const double r = allreduce(t, param[s], start[s], end[s]);
    if (s == 0 || r > red_max) red_max = r;
  }
  for (int s = 0; s + 1 < k; ++s) trans[s] = transfer(t, act[s], end[s] - 1, start[s + 1]);
  double len = (double)(m - 1) * t_max;
  len = len + (exact_floats ? py_sum(times, k) : naive_sum(times, k));
  len = len + (exact_floats ? py_sum(trans, k - 1) : naive_sum(trans, k - 1));
  len = len + red_max;
  return len;
}

// memory_feasible (pipecost.py:179-204)
__host__ __device__ inline bool memory_ok(int k, int m, const double* act, const double* param, const int* start,
                                          const int* end, double mem, double opt) {
  for (int s = 0; s < k; ++s) {
    const double n = (double)(end[s] - start[s]);
    const double act_in = s > 0 ? act[s - 1] : 0.0;
    const double ws = ((double)m * (act_in + act[s])) / n;
    if ((param[s] / n) * opt + ws > mem) return false;
  }
  return true;
}

struct PipeDev {
  int32_t F;
  const double* cost;
  const int64_t* crossing;
  const int64_t* wprefix;
  const int32_t* vprefix;
  int64_t wtotal;
  int32_t vtotal;
};

// Everything in stage_metrics after the stage sums (pipecost.py:104-141):
// scale, crossing activation bytes, parameter bytes and variable counts.
__device__ inline void stage_tail(const PipeDev& pd, const int* cuts, int P, double scale, double* comp, double* act,
                                  double* param, int* nvars) {
  int64_t wprev = 0;
  int32_t vprev = 0;
  for (int k = 0; k <= P; ++k) {
    const int64_t w = k < P ? pd.wprefix[cuts[k]] : pd.wtotal;
    const int32_t v = k < P ? pd.vprefix[cuts[k]] : pd.vtotal;
    comp[k] = comp[k] * scale;
    act[k] = k < P ? (double)pd.crossing[cuts[k]] : 0.0;
    param[k] = (double)(w - wprev);
    if (nvars) nvars[k] = v - vprev;
    wprev = w;
    vprev = v;
  }
}

// stage_metrics for sorted cut positions cuts[0..P-1] (pipecost.py:72-141).
// Costs are read through `cost` (shared or global memory).
__device__ inline void stage_metrics_dev(const PipeDev& pd, const double* cost, const int* cuts, int P, double scale,
                                         double* comp, double* act, double* param, int* nvars) {
  // One pass over the instructions; a stage closes at the first i past its
  // cut (at most one per i, as in the reference loop).  The next boundary is a
  // register so the per-instruction path is compare + load + add; lanes of a
  // warp (different candidates) stay in lockstep over i, reading the same
  // cost[i] (a shared-memory broadcast).
  int s = 0;
  int nb = P > 0 ? cuts[0] : INT_MAX;
  double acc = 0.0;
#pragma unroll 4
  for (int i = 0; i < pd.F; ++i) {
    if (i > nb) {
      comp[s] = acc;
      ++s;
      acc = 0.0;
      nb = s < P ? cuts[s] : INT_MAX;
    }
    acc = acc + cost[i];
  }
  comp[s] = acc;
  for (++s; s <= P; ++s) comp[s] = 0.0;
  stage_tail(pd, cuts, P, scale, comp, act, param, nvars);
}

// One thread per pivot tuple; the cost array is staged in shared memory when it
// fits (stage_smem), so the per-tuple sequential sums read it with broadcast loads.
__global__ void metrics_kernel(PipeDev pd, const int32_t* pivots, int64_t batch, int P, double scale, double* comp,
                               double* act, double* param, int32_t* nvars, int stage_smem) {
  pdl_entry();
  extern __shared__ double s_mcost[];
  const double* cost = pd.cost;
  if (stage_smem) {
    for (int i = threadIdx.x; i < pd.F; i += blockDim.x) s_mcost[i] = pd.cost[i];
    __syncthreads();
    cost = s_mcost;
  }
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x) {
    int cuts[kMaxStages];
    for (int k = 0; k < P; ++k) cuts[k] = pivots[b * P + k];
    double c[kMaxStages], a[kMaxStages], w[kMaxStages];
    int v[kMaxStages];
    stage_metrics_dev(pd, cost, cuts, P, scale, c, a, w, v);
    for (int k = 0; k <= P; ++k) {
      comp[b * (P + 1) + k] = c[k];
      act[b * (P + 1) + k] = a[k];
      param[b * (P + 1) + k] = w[k];
      if (nvars) nvars[b * (P + 1) + k] = v[k];
    }
  }
}

__global__ void length_kernel(Topo t, int K, int M, int64_t batch, const double* comp, const double* act,
                              const double* param, int32_t* cuts, int given, double mem, double opt, int exact,
                              double* len, uint8_t* feas) {
  pdl_entry();
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x) {
    const double* c = comp + b * K;
    const double* a = act + b * K;
    const double* w = param + b * K;
    int counts[kMaxStages], start[kMaxStages], end[kMaxStages];
    if (given) {
      int prev = 0;
      for (int s = 0; s < K; ++s) {
        const int e = s + 1 < K ? cuts[b * (K - 1) + s] : t.d;
        counts[s] = e - prev;
        prev = e;
      }
    } else {
      proportional_counts(c, K, t.d, counts);
    }
    groups_from_counts(counts, K, start, end);
    if (!given)
      for (int s = 0; s + 1 < K; ++s) cuts[b * (K - 1) + s] = end[s];
    len[b] = pipeline_len(t, K, M, c, a, w, start, end, exact != 0);
    if (feas) feas[b] = mem < 0.0 ? 1 : (memory_ok(K, M, a, w, start, end, mem, opt) ? 1 : 0);
  }
}

// candidate_pivots (pipecost.py:279-336): position i survives when the two-stage
// proportional device cut lies in the allowed set and trainables sit on both sides
__global__ void candidates_kernel(int F, const double* prefix, double total, const int32_t* cp_prefix, int32_t cp_total,
                                  Topo t, int radius, uint8_t* allowed) {
  pdl_entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < F - 1; i += gridDim.x * blockDim.x) {
    double two[2] = {prefix[i], total - prefix[i]};
    int counts[2];
    proportional_counts(two, 2, t.d, counts);
    const int cut = counts[0];
    bool ok = false;
    for (int mm = t.g; mm < t.d; mm += t.g) {  // allowed_device_cuts (pipecost.py:255-268)
      const int lo = mm - radius > 1 ? mm - radius : 1;
      const int hi = mm + radius < t.d - 1 ? mm + radius : t.d - 1;
      if (cut >= lo && cut <= hi) ok = true;
    }
    if (ok && cp_total > 0) {
      const int before = cp_prefix[i];
      if (before == 0 || before == cp_total) ok = false;
    }
    allowed[i] = ok ? 1 : 0;
  }
}

// Raw PipeTrainEnv._state features of one candidate from its stage metrics
// (envs.py:378-397): max allreduce, max transfer, min/max compute balance.
__device__ inline void train_features(const Topo& t, int K, const double* c, const double* a, const double* w,
                                      double* red_o, double* tra_o, double* bal_o, const double* fac = nullptr) {
  int counts[kMaxStages], start[kMaxStages], end[kMaxStages];
  proportional_counts(c, K, t.d, counts);
  groups_from_counts(counts, K, start, end);
  double red = 0.0, tra = 0.0, top = c[0], bot = c[0];
  for (int s = 0; s < K; ++s) {
    const double r = allreduce(t, w[s], start[s], end[s], fac);
    if (s == 0 || r > red) red = r;
    if (c[s] > top) top = c[s];
    if (c[s] < bot) bot = c[s];
  }
  for (int s = 0; s + 1 < K; ++s) {
    const double x = transfer(t, a[s], end[s] - 1, start[s + 1]);
    if (s == 0 || x > tra) tra = x;
  }
  *red_o = red;
  *tra_o = tra;
  *bal_o = top > 0.0 ? bot / top : 1.0;
}

// Per-env compaction of the action mask: list[e*C + k] = k-th allowed
// candidate of env e (ascending), count[e] = #allowed; disallowed candidates
// get their three raw features zeroed here (envs.py:386-392).  One CTA per env,
// block scan by warp ballots.
__global__ void __launch_bounds__(1024) train_compact_kernel(const uint8_t* mask, int C, int64_t E, int32_t* list,
                                                             int32_t* count, double* state) {
  pdl_entry();
  __shared__ int s_warp[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    double* st = state + e * 4 * (int64_t)C;
    int base = 0;
    for (int c0 = 0; c0 < C; c0 += blockDim.x) {
      const int i = c0 + t;
      const bool ok = i < C && mask[e * C + i] != 0;
      if (i < C && !ok) {
        st[i] = 0.0;
        st[C + i] = 0.0;
        st[2 * C + i] = 0.0;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, ok);
      if (lane == 0) s_warp[warp] = __popc(bal);
      __syncthreads();
      int off = 0, tot = 0;
      for (int w = 0; w < nwarps; ++w) {
        const int v = s_warp[w];
        off += w < warp ? v : 0;
        tot += v;
      }
      if (ok) list[e * C + base + off + __popc(bal & ((1u << lane) - 1u))] = i;
      base += tot;
      __syncthreads();
    }
    if (t == 0) count[e] = base;
  }
}

// PipeTrainEnv._state raw features.  Each thread evaluates kCandPerThread
// candidates of one env (i = chunk*128 + lane + 32*j): their stage sums run
// as interleaved add chains over one shared pass of the cost array (one
// shared-memory load and one boundary test per instruction for all chains),
// which hides the fp64 add latency and amortises the loop.  Every chain
// keeps the reference's sequential summation order, so results are
// bit-identical to the one-candidate loop.
#ifndef AP_PP_CHAINS
#define AP_PP_CHAINS 2
#endif
constexpr int kCandPerThread = AP_PP_CHAINS;
constexpr int kCandPerWarp = 32 * kCandPerThread;

__global__ void __launch_bounds__(128) train_cand_kernel(PipeDev pd, Topo t, const int32_t* cand_pos, int C,
                                                         const int32_t* applied, int A, const int32_t* list,
                                                         const int32_t* count, int64_t E, double scale,
                                                         double* state) {
  pdl_entry();
  extern __shared__ double s_cost[];
  for (int i = threadIdx.x; i < pd.F; i += blockDim.x) s_cost[i] = pd.cost[i];
  __syncthreads();
  const int nchunk = (C + kCandPerWarp - 1) / kCandPerWarp;
  const int64_t total = E * (int64_t)nchunk * 32;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = idx / (32 * (int64_t)nchunk);
    const int chunk = (int)((idx / 32) % nchunk), lane = (int)(idx % 32);
    const int n_ok = count[e];
    if (chunk * kCandPerWarp >= n_ok) continue;  // whole warp past this env's list
    double* st = state + e * 4 * (int64_t)C;
    int cand[kCandPerThread];
    bool ok[kCandPerThread];
#pragma unroll
    for (int j = 0; j < kCandPerThread; ++j) {
      const int k = chunk * kCandPerWarp + lane + 32 * j;
      ok[j] = k < n_ok;
      cand[j] = ok[j] ? list[e * C + k] : 0;
    }
    // shared applied cuts, then each chain's own candidate cut (the mask only
    // allows candidates after the last applied one, so each list is sorted)
    int acut[kMaxStages];
    int P0 = 0;
    for (int k = 0; k < A; ++k) {
      const int a = applied[e * A + k];
      if (a >= 0) acut[P0++] = cand_pos[a];
    }
    int cpos[kCandPerThread], s[kCandPerThread], nb[kCandPerThread];
    double acc[kCandPerThread];
    double comp[kCandPerThread][kMaxStages];
#pragma unroll
    for (int j = 0; j < kCandPerThread; ++j) {
      cpos[j] = ok[j] ? cand_pos[cand[j]] : INT_MAX - 1;  // idle chain: never closes
      s[j] = 0;
      nb[j] = P0 > 0 ? acut[0] : cpos[j];
      acc[j] = 0.0;
    }
    int nbmin = nb[0];
#pragma unroll
    for (int j = 1; j < kCandPerThread; ++j) nbmin = min(nbmin, nb[j]);
    const int P = P0 + 1;
    // one instruction with boundary handling (some chain closes a stage at i)
    auto step = [&](int i) {
      if (i > nbmin) {
#pragma unroll
        for (int j = 0; j < kCandPerThread; ++j) {
          if (i > nb[j]) {
            comp[j][s[j]] = acc[j];
            ++s[j];
            acc[j] = 0.0;
            nb[j] = s[j] < P0 ? acut[s[j]] : (s[j] == P0 ? cpos[j] : INT_MAX);
          }
        }
        nbmin = nb[0];
#pragma unroll
        for (int j = 1; j < kCandPerThread; ++j) nbmin = min(nbmin, nb[j]);
      }
      const double c = s_cost[i];
#pragma unroll
      for (int j = 0; j < kCandPerThread; ++j) acc[j] = acc[j] + c;
    };
    // blocks of kBlk instructions: no boundary inside -> kBlk/2 16-byte
    // shared loads from a hoisted base address and kBlk sequential adds per
    // chain (the same order as one at a time)
#ifndef AP_PP_BLOCK
#define AP_PP_BLOCK 16  // measured on B200: 16 > 8 (+4%) > 4
#endif
    constexpr int kBlk = AP_PP_BLOCK;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_cost);
    const int Fb = pd.F - pd.F % kBlk;
    int i = 0;
    for (; i < Fb; i += kBlk) {
      if (i + kBlk - 1 > nbmin) {
#pragma unroll
        for (int u = 0; u < kBlk; ++u) step(i + u);
      } else {
        double c[kBlk];
#pragma unroll
        for (int u = 0; u < kBlk; u += 2)
          asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(c[u]), "=d"(c[u + 1]) : "r"(sbase + 8u * (uint32_t)(i + u)));
#pragma unroll
        for (int u = 0; u < kBlk; ++u)
#pragma unroll
          for (int j = 0; j < kCandPerThread; ++j) acc[j] = acc[j] + c[u];
      }
    }
    for (; i < pd.F; ++i) step(i);
#pragma unroll
    for (int j = 0; j < kCandPerThread; ++j) {
      if (!ok[j]) continue;
      double* cj = comp[j];
      int sj = s[j];
      cj[sj] = acc[j];
      for (++sj; sj <= P; ++sj) cj[sj] = 0.0;
      int cuts[kMaxStages];
      for (int k = 0; k < P0; ++k) cuts[k] = acut[k];
      cuts[P0] = cpos[j];
      double a[kMaxStages], w[kMaxStages];
      stage_tail(pd, cuts, P, scale, cj, a, w, nullptr);
      double red, tra, bal;
      train_features(t, P + 1, cj, a, w, &red, &tra, &bal);
      st[cand[j]] = red;
      st[C + cand[j]] = tra;
      st[2 * C + cand[j]] = bal;
    }
  }
}

// ---- K2 with per-env reuse -------------------------------------------------
// Every allowed candidate of an env cuts after the env's last applied cut
// c_last, so its stages are: the env's fixed stages (identical for all its
// candidates), [c_last+1 .. pos] and the tail [pos+1 .. F-1].  The middle
// stage's naive sequential sum is the running sum R[pos] of one pass from
// c_last+1 (the same additions in the same order), so per candidate only the
// tail is summed.  train_prefix_kernel: one CTA per env writes fixed[e][k] and
// R[e][i]; train_tail_kernel: the candidates' tail chains + features.
__global__ void train_prefix_kernel(PipeDev pd, const int32_t* cand_pos, const int32_t* applied, int A, int64_t E,
                                    double* fixed, double* R) {
  pdl_entry();
  extern __shared__ double s_pc[];
  for (int i = threadIdx.x; i < pd.F; i += blockDim.x) s_pc[i] = pd.cost[i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    int acut[kMaxStages];
    int P0 = 0;
    for (int k = 0; k < A; ++k) {
      const int a = applied[e * A + k];
      if (a >= 0) acut[P0++] = cand_pos[a];
    }
    int i = 0;
    for (int k = 0; k < P0; ++k) {  // fixed stages [prev+1 .. acut[k]]
      double acc = 0.0;
      for (; i <= acut[k]; ++i) acc = acc + s_pc[i];
      fixed[e * kMaxStages + k] = acc;
    }
    double* __restrict__ r = R + e * (int64_t)pd.F;
    const double* __restrict__ c = s_pc;
    double acc = 0.0;  // running sum of the stage that starts at c_last + 1
    // the additions stay sequential; loads and stores are batched 8 at a time
    for (; i + 8 <= pd.F; i += 8) {
      double x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) x[u] = c[i + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        acc = acc + x[u];
        r[i + u] = acc;
      }
    }
    for (; i < pd.F; ++i) {
      acc = acc + c[i];
      r[i] = acc;
    }
  }
}

__global__ void __launch_bounds__(128) train_tail_kernel(PipeDev pd, Topo t, const int32_t* cand_pos, int C,
                                                         const int32_t* applied, int A, const int32_t* list,
                                                         const int32_t* count, int64_t E, double scale,
                                                         const double* fixed, const double* R, double* state) {
  pdl_entry();
  extern __shared__ double s_cost[];
  for (int i = threadIdx.x; i < pd.F; i += blockDim.x) s_cost[i] = pd.cost[i];
  __syncthreads();
  const int nchunk = (C + kCandPerWarp - 1) / kCandPerWarp;
  const int64_t total = E * (int64_t)nchunk * 32;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(s_cost);
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = idx / (32 * (int64_t)nchunk);
    const int chunk = (int)((idx / 32) % nchunk), lane = (int)(idx % 32);
    const int n_ok = count[e];
    if (chunk * kCandPerWarp >= n_ok) continue;  // whole warp past this env's list
    double* st = state + e * 4 * (int64_t)C;
    int cand[kCandPerThread], pos[kCandPerThread];
    bool ok[kCandPerThread];
    int lo = pd.F, hi = -1;
#pragma unroll
    for (int j = 0; j < kCandPerThread; ++j) {
      const int k = chunk * kCandPerWarp + lane + 32 * j;
      ok[j] = k < n_ok;
      cand[j] = ok[j] ? list[e * C + k] : 0;
      pos[j] = ok[j] ? cand_pos[cand[j]] : pd.F;  // idle chain: empty tail
      lo = min(lo, pos[j] + 1);
      hi = max(hi, ok[j] ? pos[j] : -1);
    }
    // tails [pos+1 .. F-1]: sequential per chain.  The warp walks one uniform
    // i (broadcast shared loads, no divergence) from its lowest start, aligned
    // down to the block; below a chain's start it adds +0.0, which leaves the
    // sum bit-identical (acc starts at +0.0 and so is never -0.0).  Blocks past
    // every start in the warp take the unconditional path.
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    double acc[kCandPerThread];
#pragma unroll
    for (int j = 0; j < kCandPerThread; ++j) acc[j] = 0.0;
    constexpr int kBlk = AP_PP_BLOCK;
    int i = lo - lo % kBlk;
    for (; i + kBlk <= pd.F && i <= hi; i += kBlk) {
      double c[kBlk];
#pragma unroll
      for (int u = 0; u < kBlk; u += 2)
        asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(c[u]), "=d"(c[u + 1]) : "r"(sbase + 8u * (uint32_t)(i + u)));
#pragma unroll
      for (int u = 0; u < kBlk; ++u)
#pragma unroll
        for (int j = 0; j < kCandPerThread; ++j) acc[j] = acc[j] + (i + u > pos[j] ? c[u] : 0.0);
    }
    for (; i + kBlk <= pd.F; i += kBlk) {
      double c[kBlk];
#pragma unroll
      for (int u = 0; u < kBlk; u += 2)
        asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(c[u]), "=d"(c[u + 1]) : "r"(sbase + 8u * (uint32_t)(i + u)));
#pragma unroll
      for (int u = 0; u < kBlk; ++u)
#pragma unroll
        for (int j = 0; j < kCandPerThread; ++j) acc[j] = acc[j] + c[u];
    }
    for (; i < pd.F; ++i) {
      const double c = s_cost[i];
#pragma unroll
      for (int j = 0; j < kCandPerThread; ++j) acc[j] = acc[j] + (i > pos[j] ? c : 0.0);
    }
    int acut[kMaxStages];
    int P0 = 0;
    for (int k = 0; k < A; ++k) {
      const int a = applied[e * A + k];
      if (a >= 0) acut[P0++] = cand_pos[a];
    }
    const int P = P0 + 1;
#pragma unroll
    for (int j = 0; j < kCandPerThread; ++j) {
      if (!ok[j]) continue;
      double cj[kMaxStages];
      for (int k = 0; k < P0; ++k) cj[k] = fixed[e * kMaxStages + k];
      cj[P0] = R[e * (int64_t)pd.F + pos[j]];
      cj[P0 + 1] = acc[j];
      int cuts[kMaxStages];
      for (int k = 0; k < P0; ++k) cuts[k] = acut[k];
      cuts[P0] = pos[j];
      double a[kMaxStages], w[kMaxStages];
      stage_tail(pd, cuts, P, scale, cj, a, w, nullptr);
      double red, tra, bal;
      train_features(t, P + 1, cj, a, w, &red, &tra, &bal);
      st[cand[j]] = red;
      st[C + cand[j]] = tra;
      st[2 * C + cand[j]] = bal;
    }
  }
}

// ---- K2 from the stage-sum table ---------------------------------------------
// Every stage of every plan the env can reach starts at 0 or just after a
// candidate cut and ends at a candidate cut or at F-1, and the cost array is
// fixed per model, so all stage sums an env ever needs form one table,
// computed once per candidate list (ap_pipe_train_table):
//   T[a][b] = naive sum of cost[start(a) .. end(b)]   (a, b in 0..C)
//   start(0) = 0, start(a) = cand_pos[a-1] + 1;  end(b) = cand_pos[b] (b < C), F-1
//   row C+1: tail[c] = T[c+1][C], the sum after cut c (contiguous for the gathers)
// Each entry is the reference's `acc = 0; acc += cost[i]` over the same
// indices in the same order (pipecost.py:72-102), so a lookup is
// bit-identical to re-summing; T[a][b] = 0.0 when the range is empty.
__global__ void train_table_kernel(PipeDev pd, const int32_t* cand_pos, int C, double* T) {
  pdl_entry();
  const int64_t W = C + 1;
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a <= C; a += gridDim.x * blockDim.x) {
    double* row = T + a * W;
    for (int b = 0; b < a; ++b) row[b] = 0.0;
    const int s = a == 0 ? 0 : cand_pos[a - 1] + 1;
    int b = a;
    double acc = 0.0;
    for (int i = s; i < pd.F && b <= C; ++i) {
      acc = acc + __ldg(pd.cost + i);
      while (b <= C && (b < C ? cand_pos[b] : pd.F - 1) <= i) row[b++] = acc;
    }
    for (; b <= C; ++b) row[b] = 0.0;  // empty ranges (start past the end)
    if (a > 0) T[W * W + (a - 1)] = row[C];
  }
}

constexpr int kFacMax = 512;  // devices covered by the table kernel's allreduce-factor table

// Per-env constants of the fixed stages (stage_tail's terms for cuts that are
// the same for every candidate of the env).
struct FixedStages {
  int P0;
  int aidx[kMaxStages];
  double comp[kMaxStages], act[kMaxStages], param[kMaxStages];
  int64_t wlast;  // wprefix at the last applied cut (0 when none)
};

// One candidate's raw features for a plan of KC stages (KC = P0 + 2 cuts + 1;
// KC == 0: the stage count Kr is a runtime value).  With KC fixed every loop
// in stage_tail / proportional_counts / train_features unrolls and the stage
// arrays live in registers.  Same operations, same order as stage_tail +
// train_features over the full cut list.
template <int KC>
__device__ __forceinline__ void cand_features(const PipeDev& pd, const Topo& t, int Kr, const FixedStages& fs,
                                              double comp_mid, double comp_tail, int64_t wp, int64_t cross,
                                              double scale, double* red, double* tra, double* bal,
                                              const double* fac) {
  constexpr int KM = KC ? KC : kMaxStages;
  const int K = KC ? KC : Kr;
  const int P0 = K - 2;
  double c[KM], a[KM], w[KM];
#pragma unroll
  for (int k = 0; k < KM; ++k)
    if (k < P0) {
      c[k] = fs.comp[k];
      a[k] = fs.act[k];
      w[k] = fs.param[k];
    }
  c[P0] = comp_mid * scale;
  a[P0] = (double)cross;
  w[P0] = (double)(wp - fs.wlast);
  c[P0 + 1] = comp_tail * scale;
  a[P0 + 1] = 0.0;
  w[P0 + 1] = (double)(pd.wtotal - wp);
  train_features(t, K, c, a, w, red, tra, bal, fac);
}

__global__ void index_positions_kernel(const int32_t* cand_pos, int C, int F, int32_t* idx_of_pos, PipeDev pd,
                                       int64_t* cand_wpre, int64_t* cand_cross) {
  pdl_entry();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const int pos = cand_pos[c];
  const bool ok = pos >= 0 && pos < F;
  if (ok) idx_of_pos[pos] = c;
  cand_wpre[c] = ok ? pd.wprefix[pos] : 0;
  cand_cross[c] = ok ? pd.crossing[pos] : 0;
}

// Batched stage_metrics from the table: a tuple whose pivots are all bound
// candidates, strictly increasing, reads its stage sums (stage k =
// T[after previous pivot][pivot k], the last T[..][C]); any other tuple takes
// the sequential sweep.  Outputs are those of metrics_kernel.
__global__ void metrics_tab_kernel(PipeDev pd, const int32_t* idx_of_pos, int C, const double* T,
                                   const int32_t* pivots, int64_t batch, int P, double scale, double* comp,
                                   double* act, double* param, int32_t* nvars) {
  pdl_entry();
  const int64_t W = C + 1;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x) {
    int cuts[kMaxStages];
    double c[kMaxStages], a[kMaxStages], w[kMaxStages];
    int v[kMaxStages];
    bool ok = true;
    int prev = -1;
    for (int k = 0; k < P; ++k) {
      const int pos = pivots[b * P + k];
      cuts[k] = pos;
      const int idx = (pos >= 0 && pos < pd.F) ? idx_of_pos[pos] : -1;
      ok = ok && idx > prev;
      if (ok) c[k] = T[(prev + 1) * W + idx];
      prev = idx;
    }
    if (ok) {
      c[P] = T[(prev + 1) * W + C];
      stage_tail(pd, cuts, P, scale, c, a, w, v);
    } else {
      stage_metrics_dev(pd, pd.cost, cuts, P, scale, c, a, w, v);
    }
    for (int k = 0; k <= P; ++k) {
      comp[b * (P + 1) + k] = c[k];
      act[b * (P + 1) + k] = a[k];
      param[b * (P + 1) + k] = w[k];
      if (nvars) nvars[b * (P + 1) + k] = v[k];
    }
  }
}

// PipeTrainEnv._state (envs.py:378-404) for E envs from the table: one CTA per
// env computes the raw features of its allowed candidates, then the block max,
// normalisation and the one-hot block -- one launch, the state written once
// and normalised from L1/L2.
template <int KC>
__device__ __forceinline__ void tab_candidates(const PipeDev& pd, const Topo& t, const int64_t* cand_wpre,
                                               const int64_t* cand_cross, int C,
                                               const double* Trow, const double* tail, const uint8_t* m,
                                               const FixedStages& fs, double scale, double* st, double& mr,
                                               double& mt, const double* fac) {
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    double red = 0.0, tra = 0.0, bal = 0.0;
    if (m[c])  // stages: fixed..., [start(alast) .. cand_pos[c]], [cand_pos[c]+1 .. F-1]
      cand_features<KC>(pd, t, fs.P0 + 2, fs, Trow[c], tail[c], cand_wpre[c], cand_cross[c], scale, &red, &tra,
                        &bal, fac);
    st[c] = red;
    st[C + c] = tra;
    st[2 * C + c] = bal;
    mr = fmax(mr, red);
    mt = fmax(mt, tra);
  }
}

#ifndef AP_PP_TAB_MINB
#define AP_PP_TAB_MINB 4  // measured on B200: 4 (64 regs) > 3 > 2 (124 regs, 25% occupancy)
#endif
__global__ void __launch_bounds__(256, AP_PP_TAB_MINB) train_state_tab_kernel(PipeDev pd, Topo t, const int32_t* cand_pos,
                                                              const int64_t* cand_wpre, const int64_t* cand_cross,
                                                              int C, const double* T, const int32_t* applied, int A,
                                                              const uint8_t* mask, int64_t E, double scale,
                                                              double* state, float* f32a, int64_t lda32,
                                                              float* f32b, int64_t ldb32) {
  pdl_entry();
  __shared__ FixedStages fs;
  __shared__ double s_max[2][32];
  __shared__ double s_fac[kFacMax + 1];  // ring allreduce factors (2(n-1))/n, n <= devices
  const int64_t W = C + 1;
  const double* tail = T + W * W;
  const double* fac = nullptr;
  if (t.d <= kFacMax) {
    for (int n = threadIdx.x; n <= t.d; n += blockDim.x) s_fac[n] = n >= 1 ? (2.0 * (double)(n - 1)) / (double)n : 0.0;
    fac = s_fac;  // published by the first barrier of the env loop
  }
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    if (threadIdx.x == 0) {
      int P0 = 0, a0 = 0;
      int64_t wprev = 0;
      for (int k = 0; k < A; ++k) {
        const int a = applied[e * A + k];
        if (a >= 0) {
          const int pos = cand_pos[a];
          const int64_t wk = pd.wprefix[pos];
          fs.aidx[P0] = a;
          fs.comp[P0] = T[a0 * W + a] * scale;  // fixed stage [start(a0) .. pos]
          fs.act[P0] = (double)pd.crossing[pos];
          fs.param[P0] = (double)(wk - wprev);
          wprev = wk;
          a0 = a + 1;
          ++P0;
        }
      }
      fs.P0 = P0;
      fs.wlast = wprev;
    }
    __syncthreads();
    const int P0 = fs.P0;
    const double* Trow = T + (P0 > 0 ? fs.aidx[P0 - 1] + 1 : 0) * W;
    double* st = state + e * 4 * (int64_t)C;
    const uint8_t* m = mask + e * (int64_t)C;
    double mr = 0.0, mt = 0.0;
    switch (P0 + 2) {  // CTA-uniform
      case 2: tab_candidates<2>(pd, t, cand_wpre, cand_cross, C, Trow, tail, m, fs, scale, st, mr, mt, fac); break;
      case 3: tab_candidates<3>(pd, t, cand_wpre, cand_cross, C, Trow, tail, m, fs, scale, st, mr, mt, fac); break;
      case 4: tab_candidates<4>(pd, t, cand_wpre, cand_cross, C, Trow, tail, m, fs, scale, st, mr, mt, fac); break;
      case 5: tab_candidates<5>(pd, t, cand_wpre, cand_cross, C, Trow, tail, m, fs, scale, st, mr, mt, fac); break;
      case 6: tab_candidates<6>(pd, t, cand_wpre, cand_cross, C, Trow, tail, m, fs, scale, st, mr, mt, fac); break;
      case 8: tab_candidates<8>(pd, t, cand_wpre, cand_cross, C, Trow, tail, m, fs, scale, st, mr, mt, fac); break;
      default: tab_candidates<0>(pd, t, cand_wpre, cand_cross, C, Trow, tail, m, fs, scale, st, mr, mt, fac); break;
    }
    for (int o = 16; o > 0; o >>= 1) {
      mr = fmax(mr, __shfl_xor_sync(0xffffffffu, mr, o));
      mt = fmax(mt, __shfl_xor_sync(0xffffffffu, mt, o));
    }
    const int wid = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
      s_max[0][wid] = mr;
      s_max[1][wid] = mt;
    }
    __syncthreads();
    mr = 0.0;
    mt = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      mr = fmax(mr, s_max[0][k]);
      mt = fmax(mt, s_max[1][k]);
    }
    for (int c = threadIdx.x; c < C; c += blockDim.x) {  // each thread re-reads its own writes
      if (mr > 0.0) st[c] = st[c] / mr;
      if (mt > 0.0) st[C + c] = st[C + c] / mt;
      double one = 0.0;
      for (int k = 0; k < P0; ++k) one = fs.aidx[k] == c ? 1.0 : one;
      st[3 * C + c] = one;
      if (f32a) {  // the learner's fp32 rows (cur / next state) straight from the same values
        const float x0 = (float)st[c], x1 = (float)st[C + c], x2 = (float)st[2 * C + c], x3 = (float)one;
        float* ra = f32a + e * lda32;
        ra[c] = x0;
        ra[C + c] = x1;
        ra[2 * C + c] = x2;
        ra[3 * C + c] = x3;
        if (f32b) {
          float* rb = f32b + e * ldb32;
          rb[c] = x0;
          rb[C + c] = x1;
          rb[2 * C + c] = x2;
          rb[3 * C + c] = x3;
        }
      }
    }
    __syncthreads();  // s_max / fs reused by the next env
  }
}

// block normalisation and one-hot (envs.py:398-404): one CTA per env
__global__ void train_norm_kernel(int C, const int32_t* applied, int A, int64_t E, double* state) {
  pdl_entry();
  __shared__ double s_max[2][32];
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    double* st = state + e * 4 * (int64_t)C;
    double mr = 0.0, mt = 0.0;
    for (int i = threadIdx.x; i < C; i += blockDim.x) {
      mr = fmax(mr, st[i]);
      mt = fmax(mt, st[C + i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
      mr = fmax(mr, __shfl_xor_sync(0xffffffffu, mr, o));
      mt = fmax(mt, __shfl_xor_sync(0xffffffffu, mt, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
      s_max[0][w] = mr;
      s_max[1][w] = mt;
    }
    __syncthreads();
    mr = 0.0;
    mt = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      mr = fmax(mr, s_max[0][k]);
      mt = fmax(mt, s_max[1][k]);
    }
    for (int i = threadIdx.x; i < C; i += blockDim.x) {
      if (mr > 0.0) st[i] = st[i] / mr;
      if (mt > 0.0) st[C + i] = st[C + i] / mt;
      st[3 * C + i] = 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int k = 0; k < A; ++k) {
        const int a = applied[e * A + k];
        if (a >= 0) st[3 * C + a] = 1.0;
      }
    __syncthreads();
  }
}

// PP-infer decode_metrics + pipeline_length (envs.py:593-616, 585)
__device__ inline double infer_point(const double* arr, int G, const Topo& t, int K, int M, const int* bnd,
                                     const int* cut) {
  const double* cc = arr;
  const double* aa = arr + G;
  const double* ww = arr + 2 * G;
  double comp[kMaxStages], act[kMaxStages], par[kMaxStages];
  int start[kMaxStages], end[kMaxStages];
  int lo = 0;
  for (int s = 0; s < K; ++s) {
    const int hi = s + 1 < K ? bnd[s] : G;
    const double c = cc[hi - 1] - (lo > 0 ? cc[lo - 1] : 0.0);
    const double w = ww[hi - 1] - (lo > 0 ? ww[lo - 1] : 0.0);
    comp[s] = c * 1000.0;
    par[s] = w;
    act[s] = hi < G ? aa[hi - 1] : 0.0;
    lo = hi;
  }
  int prev = 0;
  for (int s = 0; s < K; ++s) {
    start[s] = prev;
    end[s] = s + 1 < K ? cut[s] : t.d;
    prev = end[s];
  }
  return pipeline_len(t, K, M, comp, act, par, start, end, /*exact_floats=*/false);
}

__global__ void infer_kernel(const double* arr, int G, Topo t, int K, int M, const int32_t* bnd, const int32_t* cut,
                             int64_t batch, double* len) {
  pdl_entry();
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < batch; b += (int64_t)gridDim.x * blockDim.x) {
    int bb[kMaxStages], cc[kMaxStages];
    for (int s = 0; s + 1 < K; ++s) {
      bb[s] = bnd[b * (K - 1) + s];
      cc[s] = cut[b * (K - 1) + s];
    }
    len[b] = infer_point(arr, G, t, K, M, bb, cc);
  }
}

// exhaustive search: every (b-combo, c-combo), first-wins argmin per block
__global__ void infer_search_kernel(const double* arr, int G, Topo t, int K, int M, const int32_t* bcomb, int64_t nb,
                                    const int32_t* ccomb, int64_t nc, double* blk_len, int64_t* blk_idx) {
  pdl_entry();
  __shared__ double s_len[256];
  __shared__ int64_t s_idx[256];
  double best = INFINITY;
  int64_t best_i = INT64_MAX;
  const int64_t total = nb * nc;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ib = idx / nc, ic = idx % nc;
    int bb[kMaxStages], cc[kMaxStages];
    for (int s = 0; s + 1 < K; ++s) {
      bb[s] = bcomb[ib * (K - 1) + s];
      cc[s] = ccomb[ic * (K - 1) + s];
    }
    double l = infer_point(arr, G, t, K, M, bb, cc);
    if (l < 1e-12) l = 1e-12;  // _MIN_LENGTH (envs.py:53, 584)
    if (l < best || (l == best && idx < best_i)) {
      best = l;
      best_i = idx;
    }
  }
  s_len[threadIdx.x] = best;
  s_idx[threadIdx.x] = best_i;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      const double l2 = s_len[threadIdx.x + o];
      const int64_t i2 = s_idx[threadIdx.x + o];
      if (l2 < s_len[threadIdx.x] || (l2 == s_len[threadIdx.x] && i2 < s_idx[threadIdx.x])) {
        s_len[threadIdx.x] = l2;
        s_idx[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    blk_len[blockIdx.x] = s_len[0];
    blk_idx[blockIdx.x] = s_idx[0];
  }
}

// Table-driven exhaustive search (K <= 8 stages, <= 63 devices), bit-identical
// to infer_search_kernel.  Every division in infer_point has one operand fixed
// by the boundary combo and the other drawn from a handful of values fixed by
// the cut combo:
//   times[s] = cq[s] / n            n = group size (<= D)
//   red[s]   = (fac(n) * par[s]) / slow,  slow in {intra, inter}
//   trans[s] = act[s] / bw,         bw in {intra, inter}
// so each warp takes one boundary combo, tabulates those quotients in shared
// memory (same operands, same operations as the reference), and its lanes
// sweep the cut combos, each described by one packed word: per stage 8 bits =
// n (6) | slow is inter (1) | transfer is inter (1).
constexpr int kTabN = 64;  // table rows per stage (n = 0..63)
constexpr int kTabWarps = 8;

template <int K>
__global__ void __launch_bounds__(32 * kTabWarps) infer_search_tab_kernel(const double* arr, int G, Topo t, int M,
                                                                          const int32_t* band, const int32_t* band_off,
                                                                          int64_t nprod, const uint64_t* cword,
                                                                          int64_t nc, double* blk_len,
                                                                          int64_t* blk_idx,
                                                                          unsigned long long* n_valid) {
  pdl_entry();
  extern __shared__ double s_tab[];
  constexpr int kPerWarp = K * kTabN * 3 + 2 * K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* T = s_tab + warp * kPerWarp;  // [K][kTabN]
  double* R = T + K * kTabN;            // [K][kTabN][2]
  double* TR = R + K * kTabN * 2;       // [K][2]
  const double* cc = arr;
  const double* aa = arr + G;
  const double* ww = arr + 2 * G;
  const int nmax = t.d + 1 < kTabN ? t.d + 1 : kTabN;
  double best = INFINITY;
  int64_t best_i = INT64_MAX;
  // Boundary tuples are enumerated over the product of the per-pick bands
  // (mixed radix, last pick fastest = the host odometer's lexicographic
  // order); non-increasing tuples are skipped.  The product index ib is
  // monotone in that order, so first-wins on ib * nc + ic selects the same
  // winner as ranking the valid combos.
  for (int64_t ib = blockIdx.x * (int64_t)kTabWarps + warp; ib < nprod; ib += (int64_t)gridDim.x * kTabWarps) {
    int bnd[K];
    {
      int64_t rest = ib;
      bool inc = true;
#pragma unroll
      for (int s = K - 2; s >= 0; --s) {
        const int len = band_off[s + 1] - band_off[s];
        bnd[s] = band[band_off[s] + (int)(rest % len)];
        rest /= len;
      }
#pragma unroll
      for (int s = 1; s + 1 < K; ++s) inc &= bnd[s] > bnd[s - 1];
      if (!inc) continue;  // warp-uniform
      if (lane == 0) atomicAdd(n_valid, 1ull);
    }
    // boundary-combo metrics (infer_point's first loop)
    double cq[K], par[K], act[K];
    int lo = 0;
#pragma unroll
    for (int s = 0; s < K; ++s) {
      const int hi = s + 1 < K ? bnd[s] : G;
      const double c = cc[hi - 1] - (lo > 0 ? cc[lo - 1] : 0.0);
      const double w = ww[hi - 1] - (lo > 0 ? ww[lo - 1] : 0.0);
      cq[s] = (c * 1000.0) / 1000.0;  // comp[s] / 1000.0 as in pipeline_len
      par[s] = w;
      act[s] = hi < G ? aa[hi - 1] : 0.0;
      lo = hi;
    }
    __syncwarp();
    for (int e = lane; e < K * nmax; e += 32) {
      const int s = e / nmax, n = e % nmax;
      double q = 0.0, r0 = 0.0, r1 = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (k == s) {
          q = n >= 1 ? cq[k] / (double)n : 0.0;
          if (!(n <= 1 || par[k] == 0.0)) {  // allreduce() (topology.py:131-148)
            const double f = (2.0 * (double)(n - 1)) / (double)n;
            r0 = f * par[k] / t.intra;
            r1 = f * par[k] / t.inter;
          }
        }
      T[s * kTabN + n] = q;
      R[(s * kTabN + n) * 2 + 0] = r0;
      R[(s * kTabN + n) * 2 + 1] = r1;
    }
    if (lane < 2 * K) {
      const int s = lane >> 1;
      double a = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (k == s) a = act[k];
      TR[lane] = a / ((lane & 1) ? t.inter : t.intra);  // transfer(): bytes / bw
    }
    __syncwarp();
    for (int64_t ic = lane; ic < nc; ic += 32) {
      const uint64_t w = cword[ic];
      double times[K], tr[K];
      double t_max = 0.0, red_max = 0.0;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const uint32_t b = (uint32_t)(w >> (8 * s)) & 0xFFu;
        const int n = (int)(b & 63u);
        times[s] = T[s * kTabN + n];
        if (s == 0 || times[s] > t_max) t_max = times[s];
        const double r = R[(s * kTabN + n) * 2 + ((b >> 6) & 1u)];
        if (s == 0 || r > red_max) red_max = r;
        if (s + 1 < K) tr[s] = TR[2 * s + ((b >> 7) & 1u)];
      }
      double len = (double)(M - 1) * t_max;
      len = len + naive_sum(times, K);
      len = len + naive_sum(tr, K - 1);
      len = len + red_max;
      if (len < 1e-12) len = 1e-12;  // _MIN_LENGTH (envs.py:53, 584)
      const int64_t idx = ib * nc + ic;
      if (len < best || (len == best && idx < best_i)) {
        best = len;
        best_i = idx;
      }
    }
    __syncwarp();
  }
  // block-level first-wins argmin
  __shared__ double s_len[32 * kTabWarps];
  __shared__ int64_t s_idx[32 * kTabWarps];
  s_len[threadIdx.x] = best;
  s_idx[threadIdx.x] = best_i;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      const double l2 = s_len[threadIdx.x + o];
      const int64_t i2 = s_idx[threadIdx.x + o];
      if (l2 < s_len[threadIdx.x] || (l2 == s_len[threadIdx.x] && i2 < s_idx[threadIdx.x])) {
        s_len[threadIdx.x] = l2;
        s_idx[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    blk_len[blockIdx.x] = s_len[0];
    blk_idx[blockIdx.x] = s_idx[0];
  }
}

template <int K>
int launch_infer_tab(const double* arr, int G, const Topo& t, int M, const int32_t* d_band, const int32_t* d_off,
                     int64_t nprod, const uint64_t* d_w, int64_t nc, double* d_len, int64_t* d_idx,
                     unsigned long long* d_valid, int blocks, cudaStream_t s) {
  const size_t smem = (size_t)kTabWarps * (K * kTabN * 3 + 2 * K) * sizeof(double);
  auto k = infer_search_tab_kernel<K>;
  AP_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  launch_pdl(k, dim3(blocks), dim3(32 * kTabWarps), smem, s, arr, G, t, M, d_band, d_off, nprod, d_w, nc, d_len, d_idx, d_valid);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

Topo make_topo(const ap_topology* t) { return Topo{t->gpus_per_server, t->num_servers * t->gpus_per_server, t->intra_bw, t->inter_bw}; }

int check_topo(const ap_topology* t, int stages) {
  if (!t || t->num_servers < 1 || t->gpus_per_server < 1 || !(t->intra_bw > 0) || !(t->inter_bw > 0)) {
    set_error("invalid topology");
    return AP_ERR_INVALID;
  }
  if (stages > kMaxStages || stages < 1) {
    set_error("stage count outside [1, 32]");
    return AP_ERR_UNSUPPORTED;
  }
  return AP_OK;
}

int grid_for(int64_t n, int threads) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 148 * 16)); }

}  // namespace
}  // namespace apb

using namespace apb;

struct ap_pipe {
  int32_t F = 0;
  std::vector<double> cost, prefix;
  std::vector<int64_t> crossing, wprefix;
  std::vector<int32_t> vprefix, cp_prefix;
  int64_t wtotal = 0;
  int32_t vtotal = 0, cp_total = 0;
  double total = 0.0;
  DevBuf<double> d_cost, d_prefix;
  DevBuf<int64_t> d_crossing, d_wprefix;
  DevBuf<int32_t> d_vprefix, d_cp_prefix;
  bool uploaded = false;
  int device = 0;
  // PP-train compaction scratch (grow-only)
  int32_t* d_list = nullptr;
  int32_t* d_count = nullptr;
  int64_t list_cap = 0, count_cap = 0;

  // per-env reuse scratch: fixed stage sums [E, kMaxStages] and running sums [E, F] (grow-only)
  double* d_fixed = nullptr;
  double* d_R = nullptr;
  int64_t prefix_cap = 0;

  int ensure_prefix_scratch(int64_t n_env) {
    if (n_env > prefix_cap) {
      if (d_fixed) cudaFree(d_fixed);
      if (d_R) cudaFree(d_R);
      AP_CUDA_CHECK(cudaMalloc(&d_fixed, n_env * kMaxStages * sizeof(double)));
      AP_CUDA_CHECK(cudaMalloc(&d_R, n_env * (int64_t)std::max(F, 1) * sizeof(double)));
      prefix_cap = n_env;
    }
    return AP_OK;
  }

  // stage-sum tables bound by ap_pipe_train_table, keyed by the device
  // candidate list; kept until the handle dies (captured graphs may hold them)
  struct TableBinding {
    const int32_t* cand;
    int32_t C;
    double* tab;
    int32_t* idx_of_pos;  // [F]: candidate index at a forward position, -1 elsewhere
    int64_t* cand_wpre;   // [C]: wprefix at each candidate's position (no dependent gather per candidate)
    int64_t* cand_cross;  // [C]: crossing bytes at each candidate's position
  };
  std::vector<TableBinding> tables;
  const TableBinding* binding(const int32_t* cand, int32_t C) const {
    for (const auto& b : tables)
      if (b.cand == cand && b.C == C) return &b;
    return nullptr;
  }
  const double* table_for(const int32_t* cand, int32_t C) const {
    const TableBinding* b = binding(cand, C);
    return b ? b->tab : nullptr;
  }

  int ensure_train_scratch(int64_t n_list, int64_t n_env) {
    if (n_list > list_cap) {
      if (d_list) cudaFree(d_list);
      AP_CUDA_CHECK(cudaMalloc(&d_list, n_list * sizeof(int32_t)));
      list_cap = n_list;
    }
    if (n_env > count_cap) {
      if (d_count) cudaFree(d_count);
      AP_CUDA_CHECK(cudaMalloc(&d_count, n_env * sizeof(int32_t)));
      count_cap = n_env;
    }
    return AP_OK;
  }

  int ensure() {
    int cur = 0;
    AP_CUDA_CHECK(cudaGetDevice(&cur));
    if (uploaded) {
      if (cur != device) {
        set_error("pipe handle used on another device");
        return AP_ERR_INVALID;
      }
      return AP_OK;
    }
    device = cur;
    int rc;
    if ((rc = d_cost.upload(cost)) != AP_OK) return rc;
    if ((rc = d_prefix.upload(prefix)) != AP_OK) return rc;
    if ((rc = d_crossing.upload(crossing)) != AP_OK) return rc;
    if ((rc = d_wprefix.upload(wprefix)) != AP_OK) return rc;
    if ((rc = d_vprefix.upload(vprefix)) != AP_OK) return rc;
    if ((rc = d_cp_prefix.upload(cp_prefix)) != AP_OK) return rc;
    uploaded = true;
    return AP_OK;
  }
  PipeDev dev() const {
    return PipeDev{F, d_cost.ptr, d_crossing.ptr, d_wprefix.ptr, d_vprefix.ptr, wtotal, vtotal};
  }
  void release() {
    for (auto& b : tables) {
      cudaFree(b.tab);
      cudaFree(b.idx_of_pos);
      cudaFree(b.cand_wpre);
      cudaFree(b.cand_cross);
    }
    tables.clear();
    if (d_fixed) cudaFree(d_fixed);
    if (d_R) cudaFree(d_R);
    d_fixed = d_R = nullptr;
    prefix_cap = 0;
    if (d_list) cudaFree(d_list);
    if (d_count) cudaFree(d_count);
    d_list = d_count = nullptr;
    list_cap = count_cap = 0;
    d_cost.release();
    d_prefix.release();
    d_crossing.release();
    d_wprefix.release();
    d_vprefix.release();
    d_cp_prefix.release();
  }
};

extern "C" {

int ap_pipe_create(const ap_pipe_desc* desc, ap_pipe_t* out) {
  if (!desc || !out || desc->num_forward < 1 || desc->num_vars < 0 || !desc->cost_ms || !desc->out_bytes ||
      !desc->last_use || (desc->num_vars > 0 && (!desc->var_anchor || !desc->var_bytes))) {
    set_error("ap_pipe_create: bad descriptor");
    return AP_ERR_INVALID;
  }
  ap_pipe* p = new ap_pipe();
  const int F = desc->num_forward;
  p->F = F;
  p->cost.assign(desc->cost_ms, desc->cost_ms + F);
  // naive running prefix, exactly the reference's `acc += c` (pipecost.py:298-304)
  p->prefix.resize(F);
  double acc = 0.0;
  for (int i = 0; i < F; ++i) {
    acc += p->cost[i];
    p->prefix[i] = acc;
  }
  p->total = acc;
  // activation bytes crossing a cut after position c (pipecost.py:104-115):
  // tensor i crosses every cut in [i, last_use[i])
  std::vector<int64_t> diff(F + 1, 0);
  for (int i = 0; i < F; ++i) {
    const int lu = desc->last_use[i];
    if (lu > i) {
      diff[i] += desc->out_bytes[i];
      diff[lu] -= desc->out_bytes[i];
    }
  }
  p->crossing.resize(F);
  int64_t run = 0;
  for (int i = 0; i < F; ++i) p->crossing[i] = (run += diff[i]);
  // parameter ownership (pipecost.py:117-130): anchor -1 = stage 0 always
  std::vector<int64_t> wb(F + 1, 0);
  std::vector<int32_t> vb(F + 1, 0), cb(F + 1, 0);
  for (int v = 0; v < desc->num_vars; ++v) {
    const int a = desc->var_anchor[v];
    if (a >= F) {
      delete p;
      set_error("ap_pipe_create: var anchor out of range");
      return AP_ERR_INVALID;
    }
    wb[a < 0 ? 0 : a] += desc->var_bytes[v];
    vb[a < 0 ? 0 : a] += 1;
    p->wtotal += desc->var_bytes[v];
    p->vtotal += 1;
    if (a >= 0) {  // candidate_pivots only sees anchored variables (pipecost.py:309-319)
      cb[a] += 1;
      p->cp_total += 1;
    }
  }
  p->wprefix.resize(F);
  p->vprefix.resize(F);
  p->cp_prefix.resize(F);
  int64_t w = 0;
  int32_t vv = 0, cc = 0;
  for (int i = 0; i < F; ++i) {
    p->wprefix[i] = (w += wb[i]);
    p->vprefix[i] = (vv += vb[i]);
    p->cp_prefix[i] = (cc += cb[i]);
  }
  *out = p;
  return AP_OK;
}

int ap_pipe_destroy(ap_pipe_t p) {
  if (p) {
    p->release();
    delete p;
  }
  return AP_OK;
}

int ap_pipe_candidates(ap_pipe_t p, const ap_topology* topo, int32_t num_stages, int32_t radius, uint8_t* allowed,
                       void* stream) {
  int rc = check_topo(topo, 2);
  if (rc != AP_OK) return rc;
  if (!p || !allowed || radius < 0) {
    set_error("ap_pipe_candidates: bad arguments");
    return AP_ERR_INVALID;
  }
  if ((rc = p->ensure()) != AP_OK) return rc;
  (void)num_stages;
  const Topo t = make_topo(topo);
  launch_pdl(candidates_kernel, dim3(grid_for(p->F, 256)), dim3(256), 0, (cudaStream_t)stream, p->F, p->d_prefix.ptr, p->total,
                                                                          p->d_cp_prefix.ptr, p->cp_total, t, radius,
                                                                          allowed);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_pipe_metrics(ap_pipe_t p, const int32_t* pivots, int64_t batch, int32_t P, double bwm, double* comp,
                    double* act, double* param, int32_t* nvars, void* stream) {
  if (!p || batch < 0 || P < 0 || P + 1 > kMaxStages || (batch && (!comp || !act || !param || (P && !pivots)))) {
    set_error("ap_pipe_metrics: bad arguments");
    return AP_ERR_INVALID;
  }
  int rc = p->ensure();
  if (rc != AP_OK) return rc;
  if (batch == 0) return AP_OK;
  // small CTAs spread the (sequential-per-tuple) work over more SMs; costs in shared memory when they fit
  const size_t msmem = (size_t)p->F * sizeof(double);
  const int stage = msmem <= 200 * 1024 ? 1 : 0;
  if (stage) AP_CUDA_CHECK(cudaFuncSetAttribute(metrics_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msmem));
  launch_pdl(metrics_kernel, dim3(grid_for(batch, 32)), dim3(32), stage ? msmem : 0, (cudaStream_t)stream, p->dev(), pivots, batch, P,
                                                                                       1.0 + bwm, comp, act, param,
                                                                                       nvars, stage);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_pipe_metrics_bound(ap_pipe_t p, const int32_t* cand_pos, int32_t C, const int32_t* pivots, int64_t batch,
                          int32_t P, double bwm, double* comp, double* act, double* param, int32_t* nvars,
                          void* stream) {
  const auto* bnd = p ? p->binding(cand_pos, C) : nullptr;
  if (!bnd || std::getenv("AP_PP_NO_TABLE")) return ap_pipe_metrics(p, pivots, batch, P, bwm, comp, act, param, nvars,
                                                                     stream);
  if (batch < 0 || P < 0 || P + 1 > kMaxStages || (batch && (!comp || !act || !param || (P && !pivots)))) {
    set_error("ap_pipe_metrics_bound: bad arguments");
    return AP_ERR_INVALID;
  }
  int rc = p->ensure();
  if (rc != AP_OK) return rc;
  if (batch == 0) return AP_OK;
  launch_pdl(metrics_tab_kernel, dim3(grid_for(batch, 128)), dim3(128), 0, (cudaStream_t)stream, 
      p->dev(), bnd->idx_of_pos, C, bnd->tab, pivots, batch, P, 1.0 + bwm, comp, act, param, nvars);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_pipe_length(const ap_topology* topo, int32_t K, int32_t M, int64_t batch, const double* comp,
                   const double* act, const double* param, int32_t* cuts, int32_t given, double mem, double opt,
                   int32_t python_floats, double* len, uint8_t* feas, void* stream) {
  int rc = check_topo(topo, K);
  if (rc != AP_OK) return rc;
  if (batch < 0 || M < 1 || K > topo->num_servers * topo->gpus_per_server ||
      (batch && (!comp || !act || !param || !len || (K > 1 && !cuts)))) {
    set_error("ap_pipe_length: bad arguments");
    return AP_ERR_INVALID;
  }
  if (batch == 0) return AP_OK;
  launch_pdl(length_kernel, dim3(grid_for(batch, 128)), dim3(128), 0, (cudaStream_t)stream, make_topo(topo), K, M, batch, comp, act, param,
                                                                         cuts, given, mem, opt, python_floats, len,
                                                                         feas);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_pipe_train_table(ap_pipe_t p, const int32_t* cand_pos, int32_t C, void* stream) {
  if (!p || C < 1 || !cand_pos) {
    set_error("ap_pipe_train_table: bad arguments");
    return AP_ERR_INVALID;
  }
  int rc = p->ensure();
  if (rc != AP_OK) return rc;
  const int64_t W = (int64_t)C + 1;
  const int64_t bytes = (W * W + W) * (int64_t)sizeof(double);
  double* tab = const_cast<double*>(p->table_for(cand_pos, C));
  if (!tab) {
    if (bytes > ((int64_t)4 << 30) || p->tables.size() >= 16) {
      set_error("ap_pipe_train_table: table too large or too many bound lists (the per-candidate sweep is used)");
      return AP_ERR_UNSUPPORTED;
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    AP_CUDA_CHECK(cudaStreamIsCapturing((cudaStream_t)stream, &cs));
    if (cs != cudaStreamCaptureStatusNone) {
      set_error("ap_pipe_train_table: cannot allocate a new table during stream capture");
      return AP_ERR_INVALID;
    }
    int32_t* iop = nullptr;
    int64_t *cw = nullptr, *cx = nullptr;
    AP_CUDA_CHECK(cudaMalloc(&tab, bytes));
    AP_CUDA_CHECK(cudaMalloc(&iop, (size_t)p->F * sizeof(int32_t)));
    AP_CUDA_CHECK(cudaMalloc(&cw, (size_t)C * sizeof(int64_t)));
    AP_CUDA_CHECK(cudaMalloc(&cx, (size_t)C * sizeof(int64_t)));
    p->tables.push_back({cand_pos, C, tab, iop, cw, cx});
  }
  // (re)built from the list's current contents
  const auto* bnd = p->binding(cand_pos, C);
  launch_pdl(train_table_kernel, dim3((int)((W + 127) / 128)), dim3(128), 0, (cudaStream_t)stream, p->dev(), cand_pos, C, tab);
  AP_CUDA_CHECK(cudaGetLastError());
  AP_CUDA_CHECK(cudaMemsetAsync(bnd->idx_of_pos, 0xff, (size_t)p->F * sizeof(int32_t), (cudaStream_t)stream));
  launch_pdl(index_positions_kernel, dim3((C + 255) / 256), dim3(256), 0, (cudaStream_t)stream, cand_pos, C, p->F,
             bnd->idx_of_pos, p->dev(), bnd->cand_wpre, bnd->cand_cross);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

namespace apb {
__global__ void state_to_f32_kernel(const double* state, int64_t E, int W, float* f32a, int64_t lda32, float* f32b,
                                    int64_t ldb32) {
  pdl_entry();
  const int64_t total = E * (int64_t)W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i / W;
    const int c = (int)(i % W);
    const float x = (float)state[i];
    f32a[e * lda32 + c] = x;
    if (f32b) f32b[e * ldb32 + c] = x;
  }
}

int train_state_impl(ap_pipe_t p, const ap_topology* topo, const int32_t* cand_pos, int32_t C, const int32_t* applied,
                     int32_t A, const uint8_t* mask, int64_t E, double bwm, double* state, float* f32a, int64_t lda32,
                     float* f32b, int64_t ldb32, void* stream);
}  // namespace apb

int ap_pipe_train_state(ap_pipe_t p, const ap_topology* topo, const int32_t* cand_pos, int32_t C,
                        const int32_t* applied, int32_t A, const uint8_t* mask, int64_t E, double bwm, double* state,
                        void* stream) {
  return apb::train_state_impl(p, topo, cand_pos, C, applied, A, mask, E, bwm, state, nullptr, 0, nullptr, 0, stream);
}

int ap_pipe_train_state_ex(ap_pipe_t p, const ap_topology* topo, const int32_t* cand_pos, int32_t C,
                           const int32_t* applied, int32_t A, const uint8_t* mask, int64_t E, double bwm,
                           double* state, float* state_f32, int64_t ld_f32, float* state_f32_b, int64_t ld_f32_b,
                           void* stream) {
  if (!state_f32 || ld_f32 < 4 * (int64_t)C || (state_f32_b && ld_f32_b < 4 * (int64_t)C)) {
    set_error("ap_pipe_train_state_ex: bad fp32 outputs");
    return AP_ERR_INVALID;
  }
  return apb::train_state_impl(p, topo, cand_pos, C, applied, A, mask, E, bwm, state, state_f32, ld_f32, state_f32_b,
                          ld_f32_b, stream);
}

namespace apb {
int train_state_impl(ap_pipe_t p, const ap_topology* topo, const int32_t* cand_pos, int32_t C, const int32_t* applied,
                     int32_t A, const uint8_t* mask, int64_t E, double bwm, double* state, float* f32a, int64_t lda32,
                     float* f32b, int64_t ldb32, void* stream) {
  int rc = check_topo(topo, A + 2);
  if (rc != AP_OK) return rc;
  if (!p || C < 1 || A < 0 || E < 0 || (E && (!cand_pos || !mask || !state || (A && !applied)))) {
    set_error("ap_pipe_train_state: bad arguments");
    return AP_ERR_INVALID;
  }
  if ((rc = p->ensure()) != AP_OK) return rc;
  if (E == 0) return AP_OK;
  const Topo t = make_topo(topo);
  const auto* bnd = std::getenv("AP_PP_NO_TABLE") ? nullptr : p->binding(cand_pos, C);
  if (bnd) {  // bound candidate list: stage sums are lookups (one launch)
    launch_pdl(train_state_tab_kernel, dim3((int)std::min<int64_t>(E, 148 * 8)), dim3(256), 0, (cudaStream_t)stream,
               p->dev(), t, cand_pos, (const int64_t*)bnd->cand_wpre, (const int64_t*)bnd->cand_cross, C,
               (const double*)bnd->tab, applied, A, mask, E, 1.0 + bwm, state, f32a, lda32, f32b, ldb32);
    AP_CUDA_CHECK(cudaGetLastError());
    return AP_OK;
  }
  const size_t smem = (size_t)p->F * sizeof(double);
  if (smem > 200 * 1024) {
    set_error("ap_pipe_train_state: forward graph too long for the shared-memory cost cache "
              "(bind the candidate list with ap_pipe_train_table)");
    return AP_ERR_UNSUPPORTED;
  }
  AP_CUDA_CHECK(cudaFuncSetAttribute(train_cand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if ((rc = p->ensure_train_scratch(E * (int64_t)C, E)) != AP_OK) return rc;
  launch_pdl(train_compact_kernel, dim3((int)std::min<int64_t>(E, 148 * 4)), dim3(1024), 0, (cudaStream_t)stream, 
      mask, C, E, p->d_list, p->d_count, state);
  AP_CUDA_CHECK(cudaGetLastError());
  const int64_t threads = E * (int64_t)((C + kCandPerWarp - 1) / kCandPerWarp) * 32;
  if (std::getenv("AP_PP_FULL") == nullptr) {
    // per-env reuse: fixed stages + running sums once per env, tails per candidate
    if ((rc = p->ensure_prefix_scratch(E)) != AP_OK) return rc;
    AP_CUDA_CHECK(cudaFuncSetAttribute(train_prefix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    AP_CUDA_CHECK(cudaFuncSetAttribute(train_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(train_prefix_kernel, dim3((int)std::min<int64_t>(E, 148 * 8)), dim3(32), smem, (cudaStream_t)stream, 
        p->dev(), cand_pos, applied, A, E, p->d_fixed, p->d_R);
    AP_CUDA_CHECK(cudaGetLastError());
    launch_pdl(train_tail_kernel, dim3(grid_for(threads, 128)), dim3(128), smem, (cudaStream_t)stream, 
        p->dev(), t, cand_pos, C, applied, A, p->d_list, p->d_count, E, 1.0 + bwm, p->d_fixed, p->d_R, state);
  } else {  // one full sweep of the cost array per candidate (AP_PP_FULL=1)
    launch_pdl(train_cand_kernel, dim3(grid_for(threads, 128)), dim3(128), smem, (cudaStream_t)stream, 
        p->dev(), t, cand_pos, C, applied, A, p->d_list, p->d_count, E, 1.0 + bwm, state);
  }
  AP_CUDA_CHECK(cudaGetLastError());
  launch_pdl(train_norm_kernel, dim3((int)std::min<int64_t>(E, 148 * 8)), dim3(256), 0, (cudaStream_t)stream, C, applied, A, E, state);
  AP_CUDA_CHECK(cudaGetLastError());
  if (f32a) {
    launch_pdl(state_to_f32_kernel, dim3(grid_for(E * 4 * (int64_t)C, 256)), dim3(256), 0, (cudaStream_t)stream, state, E, 4 * C, f32a,
                                                                                          lda32, f32b, ldb32);
    AP_CUDA_CHECK(cudaGetLastError());
  }
  return AP_OK;
}
}  // namespace apb

int ap_infer_length(const double* arrays, int32_t G, const ap_topology* topo, int32_t K, int32_t M,
                    const int32_t* bnd, const int32_t* cut, int64_t batch, double* len, void* stream) {
  int rc = check_topo(topo, K);
  if (rc != AP_OK) return rc;
  if (!arrays || G < 2 || batch < 0 || (batch && (!len || (K > 1 && (!bnd || !cut))))) {
    set_error("ap_infer_length: bad arguments");
    return AP_ERR_INVALID;
  }
  if (batch == 0) return AP_OK;
  launch_pdl(infer_kernel, dim3(grid_for(batch, 128)), dim3(128), 0, (cudaStream_t)stream, arrays, G, make_topo(topo), K, M, bnd, cut,
                                                                        batch, len);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

}  // extern "C"

namespace {

// strictly increasing combinations of one value per pick, lexicographic
void combos(const int32_t* vals, const int32_t* off, int picks, std::vector<int32_t>* out) {
  std::vector<int> idx(picks, 0);
  std::vector<int32_t> cur(picks);
  out->clear();
  for (int s = 0; s < picks; ++s)
    if (off[s + 1] == off[s]) return;
  for (;;) {
    bool ok = true;
    for (int s = 0; s < picks; ++s) {
      cur[s] = vals[off[s] + idx[s]];
      if (s > 0 && cur[s] <= cur[s - 1]) ok = false;
    }
    if (ok) out->insert(out->end(), cur.begin(), cur.end());
    int s = picks - 1;
    while (s >= 0 && ++idx[s] == off[s + 1] - off[s]) idx[s--] = 0;
    if (s < 0) return;
  }
}

}  // namespace

extern "C" int ap_infer_search(const double* arrays, int32_t G, const ap_topology* topo, int32_t K, int32_t M,
                               const int32_t* band_b, const int32_t* band_b_off, const int32_t* band_c,
                               const int32_t* band_c_off, int32_t* best_b, int32_t* best_c, double* best_len,
                               int64_t* evaluated, void* stream) {
  int rc = check_topo(topo, K);
  if (rc != AP_OK) return rc;
  if (K < 2 || !arrays || !band_b || !band_b_off || !band_c || !band_c_off || !best_b || !best_c || !best_len) {
    set_error("ap_infer_search: bad arguments");
    return AP_ERR_INVALID;
  }
  const int picks = K - 1;
  std::vector<int32_t> bc, cc;
  combos(band_c, band_c_off, picks, &cc);
  const int64_t nc = (int64_t)cc.size() / picks;
  int64_t nprod = 1;  // boundary band product (the table kernel enumerates it on the device)
  for (int st = 0; st < picks; ++st) nprod *= band_b_off[st + 1] - band_b_off[st];
  cudaStream_t s = (cudaStream_t)stream;
  const Topo t = make_topo(topo);
  // packed per-cut-combo words for the table-driven kernel (see
  // infer_search_tab_kernel); any combo it cannot encode selects the general one
  std::vector<uint64_t> cw;
  bool tab = K <= 8 && t.d < kTabN && std::getenv("AP_INFER_GENERAL") == nullptr;
  if (tab) {
    cw.resize((size_t)nc);
    for (int64_t ic = 0; ic < nc && tab; ++ic) {
      uint64_t w = 0;
      int prev = 0;
      for (int st = 0; st < K && tab; ++st) {
        const int end = st + 1 < K ? cc[ic * picks + st] : t.d;
        const int n = end - prev;
        if (n < 1 || n >= kTabN) {
          tab = false;
          break;
        }
        double slow = INFINITY;  // allreduce()'s ring minimum
        for (int i = 0; i < n; ++i) slow = std::min(slow, bw(t, prev + i, prev + (i + 1) % n));
        uint64_t bits = (uint64_t)n | ((n > 1 && slow != t.intra) ? 64u : 0u);
        if (st + 1 < K) {
          const int src = end - 1, dst = end;  // transfer(end[s]-1, start[s+1])
          if (src == dst) tab = false;
          if (bw(t, src, dst) != t.intra) bits |= 128u;
        }
        w |= bits << (8 * st);
        prev = end;
      }
      if (tab) cw[(size_t)ic] = w;
    }
  }
  int64_t nb = 0;
  if (!tab) {
    combos(band_b, band_b_off, picks, &bc);
    nb = (int64_t)bc.size() / picks;
  }
  if (nc == 0 || nprod == 0 || (!tab && nb == 0)) {
    if (evaluated) *evaluated = 0;
    set_error("ap_infer_search: empty search space");
    return AP_ERR_INFEASIBLE;
  }
  int32_t *d_b = nullptr, *d_c = nullptr, *d_band = nullptr, *d_off = nullptr;
  uint64_t* d_w = nullptr;
  unsigned long long* d_valid = nullptr;
  double* d_len = nullptr;
  int64_t* d_idx = nullptr;
  const int blocks = tab ? (int)std::min<int64_t>((nprod + kTabWarps - 1) / kTabWarps, 148 * 8)
                         : (int)std::min<int64_t>((nb * nc + 255) / 256, 148 * 8);
  AP_CUDA_CHECK(cudaMalloc(&d_len, blocks * sizeof(double)));
  AP_CUDA_CHECK(cudaMalloc(&d_idx, blocks * sizeof(int64_t)));
  unsigned long long n_valid = 0;
  if (tab) {
    const int nband = band_b_off[picks];
    AP_CUDA_CHECK(cudaMalloc(&d_band, std::max(nband, 1) * sizeof(int32_t)));
    AP_CUDA_CHECK(cudaMalloc(&d_off, (picks + 1) * sizeof(int32_t)));
    AP_CUDA_CHECK(cudaMalloc(&d_valid, sizeof(unsigned long long)));
    AP_CUDA_CHECK(cudaMalloc(&d_w, cw.size() * sizeof(uint64_t)));
    AP_CUDA_CHECK(cudaMemcpyAsync(d_band, band_b, nband * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    AP_CUDA_CHECK(cudaMemcpyAsync(d_off, band_b_off, (picks + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    AP_CUDA_CHECK(cudaMemsetAsync(d_valid, 0, sizeof(unsigned long long), s));
    AP_CUDA_CHECK(cudaMemcpyAsync(d_w, cw.data(), cw.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
#define AP_TAB(KK) \
  launch_infer_tab<KK>(arrays, G, t, M, d_band, d_off, nprod, d_w, nc, d_len, d_idx, d_valid, blocks, s)
    switch (K) {
      case 2: rc = AP_TAB(2); break;
      case 3: rc = AP_TAB(3); break;
      case 4: rc = AP_TAB(4); break;
      case 5: rc = AP_TAB(5); break;
      case 6: rc = AP_TAB(6); break;
      case 7: rc = AP_TAB(7); break;
      default: rc = AP_TAB(8); break;
    }
#undef AP_TAB
    if (rc != AP_OK) return rc;
    AP_CUDA_CHECK(cudaMemcpyAsync(&n_valid, d_valid, sizeof(n_valid), cudaMemcpyDeviceToHost, s));
  } else {
    AP_CUDA_CHECK(cudaMalloc(&d_b, bc.size() * sizeof(int32_t)));
    AP_CUDA_CHECK(cudaMalloc(&d_c, cc.size() * sizeof(int32_t)));
    AP_CUDA_CHECK(cudaMemcpyAsync(d_b, bc.data(), bc.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    AP_CUDA_CHECK(cudaMemcpyAsync(d_c, cc.data(), cc.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    launch_pdl(infer_search_kernel, dim3(blocks), dim3(256), 0, s, arrays, G, t, K, M, d_b, nb, d_c, nc, d_len, d_idx);
    AP_CUDA_CHECK(cudaGetLastError());
  }
  std::vector<double> hl(blocks);
  std::vector<int64_t> hi(blocks);
  AP_CUDA_CHECK(cudaMemcpyAsync(hl.data(), d_len, blocks * sizeof(double), cudaMemcpyDeviceToHost, s));
  AP_CUDA_CHECK(cudaMemcpyAsync(hi.data(), d_idx, blocks * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  AP_CUDA_CHECK(cudaStreamSynchronize(s));
  for (void* ptr : {(void*)d_b, (void*)d_c, (void*)d_band, (void*)d_off, (void*)d_valid, (void*)d_w, (void*)d_len,
                    (void*)d_idx})
    cudaFree(ptr);
  if (tab && n_valid == 0) {
    if (evaluated) *evaluated = 0;
    set_error("ap_infer_search: empty search space");
    return AP_ERR_INFEASIBLE;
  }
  if (evaluated) *evaluated = (tab ? (int64_t)n_valid : nb) * nc;
  double bl = INFINITY;
  int64_t bi = INT64_MAX;
  for (int k = 0; k < blocks; ++k)
    if (hl[k] < bl || (hl[k] == bl && hi[k] < bi)) {
      bl = hl[k];
      bi = hi[k];
    }
  const int64_t ib = bi / nc, ic = bi % nc;
  if (tab) {  // ib is a band product index: decode it (last pick fastest)
    int64_t rest = ib;
    for (int s2 = picks - 1; s2 >= 0; --s2) {
      const int len = band_b_off[s2 + 1] - band_b_off[s2];
      best_b[s2] = band_b[band_b_off[s2] + (int)(rest % len)];
      rest /= len;
    }
  } else {
    for (int s2 = 0; s2 < picks; ++s2) best_b[s2] = bc[ib * picks + s2];
  }
  for (int s2 = 0; s2 < picks; ++s2) best_c[s2] = cc[ic * picks + s2];
  *best_len = bl;
  return AP_OK;
}
