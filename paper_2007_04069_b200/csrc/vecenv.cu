// Vectorised OPP / ADP episode driver on the device.
//
// E partition-search environments (reference PartitionSearchEnv,
// envs.py:69-230) step in lockstep without host round trips:
//   vec_apply   seeds[e, position[e]] = P or R from the chosen action
//   (K1)        batched propagation of all E seed rows
//   vec_post    reward 0.4*newP + 0.1*newR or -1 on conflict, done flags,
//               next decision position (first undecided dim in the linkage
//               order), next-state vectors, auto-reset of finished episodes
//   per_push    transitions into the device replay ring at max priority
// plus a throughput-mode PER sampler (parallel CTA scan; the parity sampler
// in dqn.cu keeps numpy's sequential order).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>

#include "engine.h"

namespace apb {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ inline uint32_t mix64to32(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return (uint32_t)x;
}

__global__ void vec_apply_kernel(int8_t* seeds, int64_t ld, const int32_t* position, const int32_t* actions, int E) {
  pdl_entry();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  seeds[(int64_t)e * ld + position[e]] = actions[e] == 0 ? 1 : 0;  // ACTION_PARTITION -> P (envs.py:45-48,137-142)
}

// one warp per env
__global__ void vec_post_kernel(int E, int n, int64_t ld, int8_t* seeds, const int8_t* status,
                                const uint8_t* outcome, const int32_t* counts, int32_t* prev_counts, int32_t* position,
                                const int32_t* order, const int32_t* order_index, float* cur_state, int64_t lds,
                                float* next_state,
                                float* rewards, uint8_t* done, uint8_t* next_mask, int A, float* ep_return,
                                float* finished_return, int32_t* finished_partitions, int32_t* episodes_done) {
  pdl_entry();
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= E) return;
  const int8_t* st = status + (int64_t)e * ld;
  float* __restrict__ cs = cur_state + (int64_t)e * lds;
  float* __restrict__ ns = next_state + (int64_t)e * lds;
  const int oc = outcome[e];
  float reward;
  bool fin;
  if (oc == AP_OUTCOME_CONFLICT) {
    reward = -1.0f;
    fin = true;
#pragma unroll 4
    for (int j = lane; j <= n; j += 32) ns[j] = cs[j];  // state unchanged (envs.py:147-149)
  } else {
    const int dP = counts[(int64_t)e * 4 + 0], dR = counts[(int64_t)e * 4 + 1];
    reward = 0.4f * (float)(dP - prev_counts[2 * e]) + 0.1f * (float)(dR - prev_counts[2 * e + 1]);
    fin = oc == AP_OUTCOME_COMPLETE;
    // next position: first undecided dim in linkage order (envs.py:207-211)
    int pos = -1;
    const int from = order_index ? order_index[position[e]] : 0;  // decided prefix of the order
    for (int base = from & ~31; base < n && pos < 0; base += 32) {
      const int j = base + lane;
      const bool und = j < n && st[order[j]] == -1;
      const unsigned bal = __ballot_sync(kFull, und);
      if (bal) pos = order[base + __ffs(bal) - 1];
    }
    // the decided statuses are the next state and the env's new current state:
    // both rows written from the same registers (no read-back of ns)
#pragma unroll 4
    for (int j = lane; j < n; j += 32) {
      const float v = (float)st[j];
      ns[j] = v;
      cs[j] = v;
    }
    if (lane == 0) {
      const float last = pos < 0 ? 1.0f : (float)pos / (float)n;
      ns[n] = last;
      cs[n] = last;
      prev_counts[2 * e] = dP;
      prev_counts[2 * e + 1] = dR;
      position[e] = pos < 0 ? 0 : pos;
    }
    if (fin && lane == 0) finished_partitions[e] = dP;
  }
  if (lane == 0) {
    rewards[e] = reward;
    done[e] = fin ? 1 : 0;
    ep_return[e] += reward;
    if (fin) {
      finished_return[e] = ep_return[e];
      if (oc == AP_OUTCOME_CONFLICT) finished_partitions[e] = -1;
      episodes_done[e] += 1;
    }
  }
  for (int j = lane; j < A; j += 32) next_mask[(int64_t)e * A + j] = fin ? 0 : 1;
  if (fin) {  // auto-reset for the next step (envs.py:103-108)
    int8_t* sd = seeds + (int64_t)e * ld;
    for (int j = lane; j < n; j += 32) {
      sd[j] = -1;
      cs[j] = -1.0f;
    }
    if (lane == 0) {
      const int first = order[0];
      cs[n] = (float)first / (float)n;
      position[e] = first;
      prev_counts[2 * e] = 0;
      prev_counts[2 * e + 1] = 0;
      ep_return[e] = 0.0f;
    }
  }
}

// Per-env incumbent of completed (non-conflict) episodes, cli.py:237-240:
// replace iff (partitions, return) is strictly greater, so within an env the
// earliest episode wins ties.  The episode id is global (step_base + e) so a
// cross-env / cross-rank reduction can keep first-wins by lowest id.
// One warp per env; the winning per-candidate status row is copied.
__global__ void vec_track_best_kernel(int E, int n, int64_t ld, const int8_t* status, const uint8_t* outcome,
                                      const uint8_t* done, const int32_t* finished_partitions,
                                      const float* finished_return, int64_t step_base, const int64_t* ctl, int world,
                                      int rank, int32_t* best_partitions, float* best_return, int64_t* best_episode,
                                      int8_t* best_status) {
  pdl_entry();
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= E || !done[e] || outcome[e] == AP_OUTCOME_CONFLICT) return;
  if (ctl) step_base = (ctl[AP_CTL_STEP] * world + rank) * (int64_t)E;
  const int32_t p = finished_partitions[e];
  const float r = finished_return[e];
  const int32_t bp = best_partitions[e];
  if (!(p > bp || (p == bp && r > best_return[e]))) return;
  const int8_t* src = status + (int64_t)e * ld;
  int8_t* dst = best_status + (int64_t)e * ld;
  for (int j = lane; j < n; j += 32) dst[j] = src[j];
  if (lane == 0) {
    best_partitions[e] = p;
    best_return[e] = r;
    best_episode[e] = step_base + e;
  }
}

__global__ void per_push_kernel(int E, int S, int A, int64_t slot0, int64_t cap, const float* states,
                                const float* next_states, int64_t lds, const int32_t* actions, const float* rewards,
                                const uint8_t* done, const uint8_t* masks, float* r_states, float* r_next,
                                int32_t* r_actions, float* r_rewards, uint8_t* r_done, uint8_t* r_masks,
                                double* r_prio, const double* max_prio, const int64_t* ctl) {
  pdl_entry();
  const int e = blockIdx.x;
  if (ctl) slot0 = ctl[AP_CTL_SLOT];
  const int64_t slot = (slot0 + e) % cap;
  // the replay ring never aliases the env's state rows: loads are batched
  // ahead of the stores (16-byte vectors when rows and bases allow)
  const float* __restrict__ s_in = states + (int64_t)e * lds;
  const float* __restrict__ n_in = next_states + (int64_t)e * lds;
  float* __restrict__ s_out = r_states + slot * S;
  float* __restrict__ n_out = r_next + slot * S;
  const bool vec = (S % 4 == 0) && (lds % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(states) | reinterpret_cast<uintptr_t>(next_states) |
                     reinterpret_cast<uintptr_t>(r_states) | reinterpret_cast<uintptr_t>(r_next)) % 16 == 0);
  if (vec) {
    const int S4 = S / 4;
    const float4* __restrict__ a = reinterpret_cast<const float4*>(s_in);
    const float4* __restrict__ b = reinterpret_cast<const float4*>(n_in);
    float4* __restrict__ ao = reinterpret_cast<float4*>(s_out);
    float4* __restrict__ bo = reinterpret_cast<float4*>(n_out);
#pragma unroll 4
    for (int j = threadIdx.x; j < S4; j += blockDim.x) {
      const float4 x = a[j], y = b[j];
      ao[j] = x;
      bo[j] = y;
    }
  } else {
#pragma unroll 4
    for (int j = threadIdx.x; j < S; j += blockDim.x) {
      const float x = s_in[j], y = n_in[j];
      s_out[j] = x;
      n_out[j] = y;
    }
  }
  for (int j = threadIdx.x; j < A; j += blockDim.x) r_masks[slot * A + j] = masks[(int64_t)e * A + j];
  if (threadIdx.x == 0) {
    r_actions[slot] = actions[e];
    r_rewards[slot] = rewards[e];
    r_done[slot] = done[e];
    r_prio[slot] = *max_prio;
  }
}

// throughput-mode PER sample over priorities already raised to alpha (kept
// scaled by ap_per_update_scaled): one 1024-thread CTA, warp-shuffle block
// scan into a CDF held in shared memory when it fits (global scratch
// otherwise), searchsorted(side='right'), IS weights normalised by the batch
// max; also refreshes the running max priority used by per_push.
// ctl != nullptr: n = ctl[AP_CTL_SIZE], uniforms from a counter hash of
// (seed, ctl[AP_CTL_TRAIN], b) instead of the `uniforms` array.
constexpr int kSampleThreads = 1024;
constexpr int kSampleSmemMax = 24576;  // doubles of CDF kept in shared memory (192 KB)

__device__ inline double warp_incl_scan(double v, int lane) {
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

__global__ void __launch_bounds__(kSampleThreads) per_sample_fast_kernel(
    const double* prio, int n, double alpha, double beta, const float* uniforms, int B, double* cdf,
    int32_t* idx_out, float* w_out, double* max_prio, const int64_t* ctl, uint64_t seed, int smem_cap) {
  pdl_entry();
  extern __shared__ double s_cdf[];
  __shared__ double w_tot[32], w_max[32];
  __shared__ float s_w[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  (void)alpha;
  uint64_t draw = 0;
  if (ctl) {
    n = (int)ctl[AP_CTL_SIZE];
    draw = (seed * 0x9E3779B97F4A7C15ULL) ^ ((uint64_t)ctl[AP_CTL_TRAIN] << 20);
    if (n < 1) {  // empty ring (caller bug): keep indices in bounds
      for (int b = t; b < B; b += kSampleThreads) {
        idx_out[b] = 0;
        w_out[b] = 0.0f;
      }
      return;
    }
  }
  double* c = n <= smem_cap ? s_cdf : cdf;
  // each warp owns a contiguous chunk, 32 elements per iteration (coalesced)
  const int chunk = ((n + 31) / 32 + 31) / 32 * 32;
  const int lo = warp * chunk, hi = min(n, lo + chunk);
  double tot = 0.0, mx = 0.0;
  int base = lo;
  for (; base + 128 <= hi; base += 128) {  // 4 loads in flight; the same per-lane accumulation order
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(prio + base + 32 * u + lane);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c[base + 32 * u + lane] = v[u];
      tot += v[u];
      mx = fmax(mx, v[u]);
    }
  }
  for (; base < hi; base += 32) {
    const int i = base + lane;
    const double v = i < hi ? prio[i] : 0.0;
    if (i < hi) c[i] = v;
    tot += v;
    mx = fmax(mx, v);
  }
  for (int o = 16; o; o >>= 1) {
    tot += __shfl_xor_sync(kFull, tot, o);
    mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  }
  if (lane == 0) {
    w_tot[warp] = tot;
    w_max[warp] = mx;
  }
  __syncthreads();
  if (warp == 0) {
    const double v = w_tot[lane];
    const double incl = warp_incl_scan(v, lane);
    w_tot[lane] = incl - v;  // exclusive offsets
    const double m = w_max[lane];
    double mm = m;
    for (int o = 16; o; o >>= 1) mm = fmax(mm, __shfl_xor_sync(kFull, mm, o));
    if (lane == 31) {
      w_max[0] = incl;  // grand total
      *max_prio = mm;
    }
  }
  __syncthreads();
  const double total = w_max[0];
  double carry = w_tot[warp];
  for (int base = lo; base < hi; base += 32) {
    const int i = base + lane;
    const double v = i < hi ? c[i] : 0.0;
    const double incl = warp_incl_scan(v, lane) + carry;
    if (i < hi) c[i] = incl;
    carry = __shfl_sync(kFull, incl, 31);
  }
  __syncthreads();
  float wm = 0.0f;
  for (int b = t; b < B; b += kSampleThreads) {
    const float ub = ctl ? (float)(mix64to32(draw + (uint64_t)b) >> 8) * (1.0f / 16777216.0f) : uniforms[b];
    const double u = (double)ub * total;
    int l = 0, h = n;
    while (l < h) {
      const int mid = (l + h) >> 1;
      if (c[mid] <= u)
        l = mid + 1;
      else
        h = mid;
    }
    if (l >= n) l = n - 1;
    idx_out[b] = l;
    const double pr = (c[l] - (l ? c[l - 1] : 0.0)) / total;
    const float w = (float)pow((double)n * pr, -beta);
    w_out[b] = w;
    wm = fmaxf(wm, w);
  }
  // normalise by the batch maximum
  for (int o = 16; o; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(kFull, wm, o));
  if (lane == 0) s_w[warp] = wm;
  __syncthreads();
  if (warp == 0) {
    float m = s_w[lane];
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
    if (lane == 0) s_w[0] = m;
  }
  __syncthreads();
  for (int b = t; b < B; b += kSampleThreads) w_out[b] /= s_w[0];
}

// Same sampler for rings whose CDF fits shared memory, with a cheaper scan:
// the CDF lives at padded index i + i/16 (conflict-free for both the coalesced
// fill and the per-thread walks); thread t sums its k = ceil(n/1024)
// contiguous priorities serially, one block scan of the thread totals gives
// the offsets, and a second serial walk writes the prefix.  (The warp-row
// kernel above runs 32 dependent warp scans per 1024 priorities.)
__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }

__global__ void __launch_bounds__(kSampleThreads) per_sample_pad_kernel(const double* prio, int n, double beta,
                                                                        const float* uniforms, int B,
                                                                        int32_t* idx_out, float* w_out,
                                                                        double* max_prio, const int64_t* ctl,
                                                                        uint64_t seed) {
  pdl_entry();
  extern __shared__ double s_c[];
  __shared__ double w_tot[32], w_max[32];
  __shared__ float s_w[32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  uint64_t draw = 0;
  if (ctl) {
    n = (int)ctl[AP_CTL_SIZE];
    draw = (seed * 0x9E3779B97F4A7C15ULL) ^ ((uint64_t)ctl[AP_CTL_TRAIN] << 20);
    if (n < 1) {  // empty ring (caller bug): keep indices in bounds
      for (int b = t; b < B; b += kSampleThreads) {
        idx_out[b] = 0;
        w_out[b] = 0.0f;
      }
      return;
    }
  }
  double mx = 0.0;
  int i = t;
  for (; i + 3 * kSampleThreads < n; i += 4 * kSampleThreads) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(prio + i + u * kSampleThreads);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s_c[pad16(i + u * kSampleThreads)] = v[u];
      mx = fmax(mx, v[u]);
    }
  }
  for (; i < n; i += kSampleThreads) {
    const double v = __ldg(prio + i);
    s_c[pad16(i)] = v;
    mx = fmax(mx, v);
  }
  __syncthreads();
  const int k = (n + kSampleThreads - 1) / kSampleThreads;
  const int lo = min(n, t * k), hi = min(n, lo + k);
  double tot = 0.0;
  for (int j = lo; j < hi; ++j) tot += s_c[pad16(j)];
  const double incl = warp_incl_scan(tot, lane);
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  if (lane == 31) w_tot[warp] = incl;
  if (lane == 0) w_max[warp] = mx;
  __syncthreads();
  if (warp == 0) {
    const double v = w_tot[lane];
    const double wi = warp_incl_scan(v, lane);
    w_tot[lane] = wi - v;  // exclusive warp offsets
    double mm = w_max[lane];
    for (int o = 16; o; o >>= 1) mm = fmax(mm, __shfl_xor_sync(kFull, mm, o));
    if (lane == 31) {
      w_max[0] = wi;  // grand total
      *max_prio = mm;
    }
  }
  __syncthreads();
  double run = (incl - tot) + w_tot[warp];
  for (int j = lo; j < hi; ++j) {
    run += s_c[pad16(j)];
    s_c[pad16(j)] = run;
  }
  __syncthreads();
  const double total = w_max[0];
  float wm = 0.0f;
  for (int b = t; b < B; b += kSampleThreads) {
    const float ub = ctl ? (float)(mix64to32(draw + (uint64_t)b) >> 8) * (1.0f / 16777216.0f) : uniforms[b];
    const double u = (double)ub * total;
    int l = 0, h = n;
    while (l < h) {
      const int mid = (l + h) >> 1;
      if (s_c[pad16(mid)] <= u)
        l = mid + 1;
      else
        h = mid;
    }
    if (l >= n) l = n - 1;
    idx_out[b] = l;
    const double pr = (s_c[pad16(l)] - (l ? s_c[pad16(l - 1)] : 0.0)) / total;
    const float w = (float)pow((double)n * pr, -beta);
    w_out[b] = w;
    wm = fmaxf(wm, w);
  }
  for (int o = 16; o; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(kFull, wm, o));
  if (lane == 0) s_w[warp] = wm;
  __syncthreads();
  if (warp == 0) {
    float m = s_w[lane];
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
    if (lane == 0) s_w[0] = m;
  }
  __syncthreads();
  for (int b = t; b < B; b += kSampleThreads) w_out[b] /= s_w[0];
}

int launch_per_sample(const double* prio, int n_host_max, double beta, const float* uniforms, int B, double* cdf,
                      int32_t* idx, float* w, double* max_prio, const int64_t* ctl, uint64_t seed, cudaStream_t s) {
  if (n_host_max <= kSampleSmemMax && std::getenv("AP_PER_ROWSCAN") == nullptr) {  // padded CDF in shared memory
    const int64_t psmem = (int64_t)(n_host_max + n_host_max / 16 + 1) * 8;
    static PerDeviceMax pconfigured;
    if (pconfigured.need(current_device(), psmem + 1))
      AP_CUDA_CHECK(cudaFuncSetAttribute(per_sample_pad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)psmem));
    launch_pdl(per_sample_pad_kernel, dim3(1), dim3(kSampleThreads), (size_t)psmem, s, prio, n_host_max, beta,
               uniforms, B, idx, w, max_prio, ctl, seed);
    AP_CUDA_CHECK(cudaGetLastError());
    return AP_OK;
  }
  // shared CDF sized for the largest ring this launch can see
  const int64_t smem = n_host_max <= kSampleSmemMax ? (int64_t)n_host_max * 8 : 0;
  static PerDeviceMax configured;
  if (configured.need(current_device(), smem + 1))
    AP_CUDA_CHECK(cudaFuncSetAttribute(per_sample_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::max<int64_t>(smem, 0)));
  launch_pdl(per_sample_fast_kernel, dim3(1), dim3(kSampleThreads), (size_t)smem, s, prio, n_host_max, 0.0, beta, uniforms, B, cdf, idx, w,
                                                                 max_prio, ctl, seed, (int)(smem / 8));
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

// ---- vectorised PipeTrainEnv (envs.py:276-404) --------------------------------
// picks [E, P] (P = K - 1 candidate indices), positions [E, P] (their forward
// positions, pre-filled with valid dummies so every row is a legal pivot tuple
// for the batched metrics kernel), n_applied [E].
__global__ void vec_pipe_apply_kernel(int E, int P, const int32_t* actions, const int32_t* cand_pos, int32_t* picks,
                                      int32_t* positions, int32_t* n_applied, uint8_t* done) {
  pdl_entry();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int k = n_applied[e];
  const int a = actions[e];
  picks[(int64_t)e * P + k] = a;
  positions[(int64_t)e * P + k] = cand_pos[a];
  n_applied[e] = k + 1;
  done[e] = (k + 1 == P) ? 1 : 0;
}

// Terminal rewards (1 / L, 1 / sqrt L, -1 / sqrt L when infeasible), per-env
// incumbents (min L over feasible episodes, strict <: cli.py:315), reset of
// finished envs, then the state inputs of every env: the applied picks (first
// a_max) and the action mask (envs.py:284-293); next_mask = 0 for finished envs.
__global__ void vec_pipe_post_kernel(int E, int C, int P, int a_max, const double* length, const uint8_t* feasible,
                                     const uint8_t* done, int reward_shape, const int32_t* dummy_pos, float* rewards,
                                     int32_t* picks, int32_t* positions, int32_t* n_applied, int32_t* applied_state,
                                     uint8_t* mask, uint8_t* next_mask, double* best_len, int32_t* best_picks,
                                     int64_t* best_episode, float* ep_return, float* finished_return,
                                     int32_t* episodes_done, const int64_t* ctl, int world, int rank) {
  pdl_entry();
  const int e = blockIdx.x;
  const bool fin = done[e] != 0;
  const int64_t step_base = (ctl[AP_CTL_STEP] * world + rank) * (int64_t)E;
  __shared__ int s_k, s_last;
  if (threadIdx.x == 0) {
    float r = 0.0f;
    if (fin) {
      const double L = fmax(length[e], 1e-12);  // _MIN_LENGTH
      const bool feas = feasible[e] != 0;
      r = !feas ? (float)(-1.0 / sqrt(L)) : (reward_shape == 0 ? (float)(1.0 / L) : (float)(1.0 / sqrt(L)));
      if (feas && L < best_len[e]) {
        best_len[e] = L;
        for (int k = 0; k < P; ++k) best_picks[(int64_t)e * P + k] = picks[(int64_t)e * P + k];
        best_episode[e] = step_base + e;
      }
      finished_return[e] = ep_return[e] + r;
      ep_return[e] = 0.0f;
      episodes_done[e] += 1;
      n_applied[e] = 0;  // auto-reset (envs.py:275-278)
      for (int k = 0; k < P; ++k) {
        picks[(int64_t)e * P + k] = -1;
        positions[(int64_t)e * P + k] = dummy_pos[k];
      }
    } else {
      ep_return[e] += r;
    }
    rewards[e] = r;
    const int k = n_applied[e];
    s_k = k;
    s_last = k > 0 ? picks[(int64_t)e * P + k - 1] : -1;
    for (int j = 0; j < a_max; ++j) applied_state[(int64_t)e * a_max + j] = j < k ? picks[(int64_t)e * P + j] : -1;
  }
  __syncthreads();
  const int remaining = P - s_k;
  const int hi = C - remaining;  // keep room for the picks still owed
  for (int i = threadIdx.x; i < C; i += blockDim.x) {
    const uint8_t m = (i > s_last && i <= hi) ? 1 : 0;
    mask[(int64_t)e * C + i] = m;
    next_mask[(int64_t)e * C + i] = fin ? 0 : m;
  }
}

// ---- vectorised PipeInferEnv (envs.py:407-626) --------------------------------
// bnd / cut [E, P] boundaries in 1..G-1 and device cuts in 1..D-1 (dummy tails keep
// every row a legal point for the batched length kernel), nb / nc [E] counts.
__global__ void vec_infer_apply_kernel(int E, int P, int G, const int32_t* actions, int32_t* bnd, int32_t* cut,
                                       int32_t* nb, int32_t* nc, uint8_t* done) {
  pdl_entry();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int a = actions[e];
  if (a < G - 1) {
    bnd[(int64_t)e * P + nb[e]] = a + 1;
    nb[e] += 1;
  } else {
    cut[(int64_t)e * P + nc[e]] = a - (G - 1) + 1;
    nc[e] += 1;
  }
  done[e] = nc[e] == P ? 1 : 0;
}

// Terminal rewards 1 / max(L, 1e-12), incumbents (min L, strict <), reset,
// the phased action mask (boundaries, then cuts, each increasing and leaving
// room for the picks still owed, within the per-pick bands: envs.py:447-469)
// and the pick slots of the state (b / G, c / D after the static part).
__global__ void vec_infer_post_kernel(int E, int P, int G, int D, int S, int64_t lds, const double* length,
                                      const uint8_t* done,
                                      const int32_t* dummy_b, const int32_t* dummy_c, const uint8_t* band_b,
                                      const uint8_t* band_c, float* rewards, int32_t* bnd, int32_t* cut,
                                      int32_t* nb, int32_t* nc, uint8_t* mask, uint8_t* next_mask, float* state,
                                      double* best_len, int32_t* best_b, int32_t* best_c, int64_t* best_episode,
                                      float* ep_return, float* finished_return, int32_t* episodes_done,
                                      const int64_t* ctl, int world, int rank) {
  pdl_entry();
  const int e = blockIdx.x;
  const bool fin = done[e] != 0;
  __shared__ int s_nb, s_nc, s_lb, s_lc;
  if (threadIdx.x == 0) {
    float r = 0.0f;
    if (fin) {
      const double L = fmax(length[e], 1e-12);
      r = (float)(1.0 / L);
      if (L < best_len[e]) {
        best_len[e] = L;
        for (int k = 0; k < P; ++k) {
          best_b[(int64_t)e * P + k] = bnd[(int64_t)e * P + k];
          best_c[(int64_t)e * P + k] = cut[(int64_t)e * P + k];
        }
        best_episode[e] = (ctl[AP_CTL_STEP] * world + rank) * (int64_t)E + e;
      }
      finished_return[e] = ep_return[e] + r;
      ep_return[e] = 0.0f;
      episodes_done[e] += 1;
      nb[e] = 0;
      nc[e] = 0;
      for (int k = 0; k < P; ++k) {
        bnd[(int64_t)e * P + k] = dummy_b[k];
        cut[(int64_t)e * P + k] = dummy_c[k];
      }
    } else {
      ep_return[e] += r;
    }
    rewards[e] = r;
    s_nb = nb[e];
    s_nc = nc[e];
    s_lb = s_nb > 0 ? bnd[(int64_t)e * P + s_nb - 1] : 0;
    s_lc = s_nc > 0 ? cut[(int64_t)e * P + s_nc - 1] : 0;
    float* slots = state + (int64_t)e * lds + (S - 2 * P);
    for (int k = 0; k < P; ++k) {
      slots[k] = k < s_nb ? (float)((double)bnd[(int64_t)e * P + k] / (double)G) : 0.0f;
      slots[P + k] = k < s_nc ? (float)((double)cut[(int64_t)e * P + k] / (double)D) : 0.0f;
    }
  }
  __syncthreads();
  const int A = (G - 1) + (D - 1);
  const bool bphase = s_nb < P;
  for (int j = threadIdx.x; j < A; j += blockDim.x) {
    uint8_t m = 0;
    if (bphase && j < G - 1) {
      const int b = j + 1;
      m = b > s_lb && b <= G - (P - s_nb) && band_b[(int64_t)s_nb * G + b];
    } else if (!bphase && j >= G - 1) {
      const int c = j - (G - 1) + 1;
      m = c > s_lc && c <= D - (P - s_nc) && band_c[(int64_t)s_nc * D + c];
    }
    mask[(int64_t)e * A + j] = m;
    next_mask[(int64_t)e * A + j] = fin ? 0 : m;
  }
}

// mode 0: one learn step done (train counter); mode 1: one vector step done
// (step counter, ring slot and size after pushing E transitions)
__global__ void ctl_advance_kernel(int64_t* ctl, int mode, int64_t E, int64_t cap) {
  pdl_entry();
  if (mode == 0) {
    ctl[AP_CTL_TRAIN] += 1;
  } else {
    ctl[AP_CTL_STEP] += 1;
    ctl[AP_CTL_SLOT] = (ctl[AP_CTL_SLOT] + E) % cap;
    ctl[AP_CTL_SIZE] = ctl[AP_CTL_SIZE] + E < cap ? ctl[AP_CTL_SIZE] + E : cap;
  }
}

// scaled[idx] = (|td| + 1e-6)**alpha, last duplicate wins
// ctl != nullptr: also counts the finished learn step (ctl[AP_CTL_TRAIN] += 1)
__global__ void per_update_scaled_kernel(double* scaled, const int32_t* idx, const float* td, int B, double alpha,
                                         int64_t* ctl) {
  pdl_entry();
  __shared__ int32_t s_idx[1024];  // the batch's indices for the duplicate scan (B <= 1024)
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (ctl && b == 0) ctl[AP_CTL_TRAIN] += 1;
  const bool staged = B <= 1024;
  if (staged) {
    for (int k = threadIdx.x; k < B; k += blockDim.x) s_idx[k] = idx[k];
    __syncthreads();
  }
  if (b >= B) return;
  const int32_t* ix = staged ? s_idx : idx;
  const int32_t mine = ix[b];
  for (int k = b + 1; k < B; ++k)  // last write wins (agent.py:224-226)
    if (ix[k] == mine) return;
  scaled[mine] = pow(fabs((double)td[b]) + 1e-6, alpha);
}

}  // namespace
}  // namespace apb

using namespace apb;

extern "C" {

int ap_vec_apply(int8_t* seeds, int64_t ld, const int32_t* position, const int32_t* actions, int32_t E, void* stream) {
  if (E <= 0) return AP_OK;
  launch_pdl(vec_apply_kernel, dim3((E + 255) / 256), dim3(256), 0, (cudaStream_t)stream, seeds, ld, position, actions, E);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_vec_post(int32_t E, int32_t n, int64_t ld, int8_t* seeds, const int8_t* status, const uint8_t* outcome,
                const int32_t* counts, int32_t* prev_counts, int32_t* position, const int32_t* order,
                const int32_t* order_index, float* cur_state,
                int64_t lds, float* next_state, float* rewards, uint8_t* done, uint8_t* next_mask, int32_t A,
                float* ep_return, float* finished_return, int32_t* finished_partitions, int32_t* episodes_done,
                void* stream) {
  if (E <= 0) return AP_OK;
  launch_pdl(vec_post_kernel, dim3((E + 7) / 8), dim3(256), 0, (cudaStream_t)stream, 
      E, n, ld, seeds, status, outcome, counts, prev_counts, position, order, order_index, cur_state, lds, next_state,
      rewards, done,
      next_mask, A, ep_return, finished_return, finished_partitions, episodes_done);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_vec_track_best(int32_t E, int32_t n, int64_t ld, const int8_t* status, const uint8_t* outcome,
                      const uint8_t* done, const int32_t* finished_partitions, const float* finished_return,
                      int64_t step_base, const int64_t* ctl, int32_t world, int32_t rank, int32_t* best_partitions,
                      float* best_return, int64_t* best_episode, int8_t* best_status, void* stream) {
  if (E <= 0) return AP_OK;
  if (ctl && (world < 1 || rank < 0 || rank >= world)) {
    set_error("ap_vec_track_best: bad world / rank");
    return AP_ERR_INVALID;
  }
  launch_pdl(vec_track_best_kernel, dim3((E + 7) / 8), dim3(256), 0, (cudaStream_t)stream, 
      E, n, ld, status, outcome, done, finished_partitions, finished_return, step_base, ctl, world, rank,
      best_partitions, best_return, best_episode, best_status);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_per_push(int32_t E, int32_t S, int32_t A, int64_t slot0, int64_t cap, const float* states,
                const float* next_states, int64_t lds, const int32_t* actions, const float* rewards,
                const uint8_t* done, const uint8_t* masks, float* r_states, float* r_next, int32_t* r_actions,
                float* r_rewards, uint8_t* r_done, uint8_t* r_masks, double* r_prio, const double* max_prio,
                void* stream) {
  if (E <= 0) return AP_OK;
  launch_pdl(per_push_kernel, dim3(E), dim3(128), 0, (cudaStream_t)stream, E, S, A, slot0, cap, states, next_states, lds, actions, rewards,
                                                       done, masks, r_states, r_next, r_actions, r_rewards, r_done,
                                                       r_masks, r_prio, max_prio, nullptr);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_per_push_ctl(int32_t E, int32_t S, int32_t A, int64_t cap, const float* states, const float* next_states,
                    int64_t lds, const int32_t* actions, const float* rewards, const uint8_t* done,
                    const uint8_t* masks, float* r_states, float* r_next, int32_t* r_actions, float* r_rewards,
                    uint8_t* r_done, uint8_t* r_masks, double* r_prio, const double* max_prio, const int64_t* ctl,
                    void* stream) {
  if (!ctl || cap < 1) {
    set_error("ap_per_push_ctl: bad arguments");
    return AP_ERR_INVALID;
  }
  if (E <= 0) return AP_OK;
  launch_pdl(per_push_kernel, dim3(E), dim3(128), 0, (cudaStream_t)stream, E, S, A, 0, cap, states, next_states, lds, actions, rewards,
                                                       done, masks, r_states, r_next, r_actions, r_rewards, r_done,
                                                       r_masks, r_prio, max_prio, ctl);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_per_sample_fast(const double* priorities, int32_t n, double alpha, double beta, const float* uniforms, int32_t B,
                       double* cdf_scratch, int32_t* indices, float* weights, double* max_priority, void* stream) {
  if (n < 1 || B < 1) {
    set_error("ap_per_sample_fast: empty buffer or batch");
    return AP_ERR_INVALID;
  }
  (void)alpha;  // priorities are kept raised to alpha
  return launch_per_sample(priorities, n, beta, uniforms, B, cdf_scratch, indices, weights, max_priority, nullptr, 0,
                           (cudaStream_t)stream);
}

int ap_per_sample_ctl(const double* priorities, int64_t capacity, double beta, int32_t B, uint64_t seed,
                      double* cdf_scratch, int32_t* indices, float* weights, double* max_priority, const int64_t* ctl,
                      void* stream) {
  if (!ctl || B < 1 || capacity < 1 || capacity > INT32_MAX) {
    set_error("ap_per_sample_ctl: bad arguments");
    return AP_ERR_INVALID;
  }
  return launch_per_sample(priorities, (int)capacity, beta, nullptr, B, cdf_scratch, indices, weights, max_priority,
                           ctl, seed, (cudaStream_t)stream);
}

int ap_vec_pipe_apply(int32_t E, int32_t P, const int32_t* actions, const int32_t* cand_pos, int32_t* picks,
                      int32_t* positions, int32_t* n_applied, uint8_t* done, void* stream) {
  if (E < 0 || P < 1 || (E > 0 && (!actions || !cand_pos || !picks || !positions || !n_applied || !done))) {
    set_error("ap_vec_pipe_apply: bad arguments");
    return AP_ERR_INVALID;
  }
  if (E == 0) return AP_OK;
  launch_pdl(vec_pipe_apply_kernel, dim3((E + 255) / 256), dim3(256), 0, (cudaStream_t)stream, E, P, actions, cand_pos, picks, positions,
                                                                           n_applied, done);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_vec_pipe_post(int32_t E, int32_t C, int32_t P, int32_t a_max, const double* length, const uint8_t* feasible,
                     const uint8_t* done, int32_t reward_shape, const int32_t* dummy_pos, float* rewards,
                     int32_t* picks, int32_t* positions, int32_t* n_applied, int32_t* applied_state, uint8_t* mask,
                     uint8_t* next_mask, double* best_len, int32_t* best_picks, int64_t* best_episode,
                     float* ep_return, float* finished_return, int32_t* episodes_done, const int64_t* ctl,
                     int32_t world, int32_t rank, void* stream) {
  if (E < 0 || C < 1 || P < 1 || a_max < 1 || (reward_shape != 0 && reward_shape != 1) || !ctl || world < 1 ||
      rank < 0 || rank >= world) {
    set_error("ap_vec_pipe_post: bad arguments");
    return AP_ERR_INVALID;
  }
  if (E == 0) return AP_OK;
  // one CTA per env; episodes finishing at this step get global ids (step * world + rank) * E + e
  launch_pdl(vec_pipe_post_kernel, dim3(E), dim3(128), 0, (cudaStream_t)stream, 
      E, C, P, a_max, length, feasible, done, reward_shape, dummy_pos, rewards, picks, positions, n_applied,
      applied_state, mask, next_mask, best_len, best_picks, best_episode, ep_return, finished_return, episodes_done,
      ctl, world, rank);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_vec_infer_apply(int32_t E, int32_t P, int32_t G, const int32_t* actions, int32_t* bnd, int32_t* cut,
                       int32_t* nb, int32_t* nc, uint8_t* done, void* stream) {
  if (E < 0 || P < 1 || G < 2 || (E > 0 && (!actions || !bnd || !cut || !nb || !nc || !done))) {
    set_error("ap_vec_infer_apply: bad arguments");
    return AP_ERR_INVALID;
  }
  if (E == 0) return AP_OK;
  launch_pdl(vec_infer_apply_kernel, dim3((E + 255) / 256), dim3(256), 0, (cudaStream_t)stream, E, P, G, actions, bnd, cut, nb, nc, done);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_vec_infer_post(int32_t E, int32_t P, int32_t G, int32_t D, int32_t S, int64_t ld_state, const double* length,
                      const uint8_t* done, const int32_t* dummy_b, const int32_t* dummy_c, const uint8_t* band_b,
                      const uint8_t* band_c, float* rewards, int32_t* bnd, int32_t* cut, int32_t* nb, int32_t* nc,
                      uint8_t* mask, uint8_t* next_mask, float* state, double* best_len, int32_t* best_b,
                      int32_t* best_c, int64_t* best_episode, float* ep_return, float* finished_return,
                      int32_t* episodes_done, const int64_t* ctl, int32_t world, int32_t rank, void* stream) {
  if (E < 0 || P < 1 || G < 2 || D < 2 || S < 2 * P || ld_state < S || !ctl || world < 1 || rank < 0 ||
      rank >= world) {
    set_error("ap_vec_infer_post: bad arguments");
    return AP_ERR_INVALID;
  }
  if (E == 0) return AP_OK;
  launch_pdl(vec_infer_post_kernel, dim3(E), dim3(128), 0, (cudaStream_t)stream, 
      E, P, G, D, S, ld_state, length, done, dummy_b, dummy_c, band_b, band_c, rewards, bnd, cut, nb, nc, mask,
      next_mask, state,
      best_len, best_b, best_c, best_episode, ep_return, finished_return, episodes_done, ctl, world, rank);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_vec_ctl_advance(int64_t* ctl, int32_t mode, int64_t E, int64_t cap, void* stream) {
  if (!ctl || (mode != 0 && mode != 1) || cap < 1) {
    set_error("ap_vec_ctl_advance: bad arguments");
    return AP_ERR_INVALID;
  }
  launch_pdl(ctl_advance_kernel, dim3(1), dim3(1), 0, (cudaStream_t)stream, ctl, mode, E, cap);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_per_update_scaled(double* scaled, const int32_t* indices, const float* td, int32_t B, double alpha,
                         void* stream) {
  if (B <= 0) return AP_OK;
  launch_pdl(per_update_scaled_kernel, dim3((B + 127) / 128), dim3(128), 0, (cudaStream_t)stream, scaled, indices, td, B, alpha,
                                                                             nullptr);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_per_update_scaled_ctl(double* scaled, const int32_t* indices, const float* td, int32_t B, double alpha,
                             int64_t* ctl, void* stream) {
  if (!ctl || B < 1) {
    set_error("ap_per_update_scaled_ctl: bad arguments");
    return AP_ERR_INVALID;
  }
  launch_pdl(per_update_scaled_kernel, dim3((B + 127) / 128), dim3(128), 0, (cudaStream_t)stream, scaled, indices, td, B, alpha, ctl);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

}  // extern "C"
