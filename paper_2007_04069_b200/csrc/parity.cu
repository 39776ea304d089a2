// Reference-semantics search loop on the device (parity mode, one environment).
//
// The reference episode loop `train_partition` (cli.py:193-248) runs, per step,
// agent.act (agent.py:155-170: numpy PCG64 random() then, when exploring,
// integers(#allowed); else masked argmax of Q), env.step (envs.py:133-175: seed
// the dim up for decision, re-propagate, reward 0.4 * #new P + 0.1 * #new R or
// -1 on CONFLICT, next position in the linkage order), agent.observe (push with
// the current max priority, agent.py:197-205) and agent.learn (PER sample from
// 64 more random() draws, double-DQN update, Adam, priorities, target sync every
// 100 train steps, agent.py:207-337).  Here every one of those runs on the GPU.  With the
// fused learner (devloop.py) one step of the loop body is
//
//   ap_parity_sample (early mode) ----------------------------------------.
//   ap_parity_act_fused -> K1 (one row) -> ap_parity_post ----------------+-> ap_dqn_learn_fused
//
// (the sampler replays the act's draws and counts the pending push, so it runs beside the env
// kernels; the act skips its forward on exploring steps; the learn kernel keeps the loss log,
// train counter, target sync and the PER caches), 8 such steps form the body of a WHILE node
// (episodes done < budget).  With the tensor-core GEMM learner the body is the step graph
// forward -> ap_parity_act -> K1 -> ap_parity_post and an IF (ring >= batch) node holding
// sample (late mode) -> learn GEMMs -> ap_parity_learn_tail -> ap_parity_target_sync.
// Nothing returns to the host until the episode budget is spent.  The random
// stream is numpy's own (pcg64.cuh), so draws, actions, rewards, states and the
// chosen plan are those of the host-driven loop bit for bit
// (tests/test_devloop_gpu.py).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <new>

#include "engine.h"

#ifdef AP_SAMPLE_TRACE  // dev-only: SM clock at the sampler's stages (thread 0; one CTA, one SM)
__device__ unsigned long long g_sample_trace[16];
extern "C" int ap_debug_sample_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_sample_trace, sizeof(g_sample_trace));
}
#define ST(k)                                                          \
  do {                                                                 \
    if (threadIdx.x == 0) {                                            \
      unsigned long long t_;                                           \
      t_ = clock64();                                                  \
      g_sample_trace[k] = t_;                                          \
    }                                                                  \
  } while (0)
#endif

#include "parity_act.cuh"
#include "pcg64.cuh"
#include "per_sample.cuh"

namespace apb {
namespace {

constexpr int kPostThreads = 256;
constexpr int kSampleMaxB = 1024;

// state row entry of the decision position: flat index / |D| in fp64, stored as fp32
// (the host agent converts the fp64 state to fp32 the same way); 1.0 when no position
__device__ __forceinline__ float position_feature(int64_t pos, int n) {
  return pos < 0 ? 1.0f : (float)__ddiv_rn((double)pos, (double)n);
}

__global__ void __launch_bounds__(kPostThreads) parity_act_kernel(ap_parity_loop L, const float* __restrict__ q,
                                                                  int32_t* __restrict__ action) {
  pdl_entry();
  __syncthreads();  // every thread has read the control block before thread 0 writes to it
  parity_step_begin(L, false, threadIdx.x == 0);
  parity_act_rows(L);
  __syncthreads();
  if (threadIdx.x == 0) parity_act_decide(L, q, action);
}

__device__ __forceinline__ int block_sum(int v, int* s_red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
  __syncthreads();
  return t;
}

__device__ __forceinline__ int block_min(int v, int* s_red) {
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = v;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = min(t, s_red[w]);
  __syncthreads();
  return t;
}

// env.step post-processing + episode bookkeeping + agent.observe, one CTA
__global__ void __launch_bounds__(kPostThreads) parity_post_kernel(ap_parity_loop L, const int32_t* __restrict__ action) {
  pdl_entry();
  if (!L.ctl[AP_PL_ACTIVE]) return;  // the budget ran out earlier in this WHILE iteration
  __shared__ int s_red[kPostThreads / 32];
  __shared__ double s_prio[kPostThreads / 32];
  const int n = L.n;
  const int tid = threadIdx.x;
  const uint8_t oc = *L.outcome;
  const bool conflict = oc == AP_OUTCOME_CONFLICT;
  const bool complete = oc == AP_OUTCOME_COMPLETE;
  const int64_t step = L.ctl[AP_PL_STEP];
  const int64_t slot = L.ctl[AP_CTL_SLOT], size = L.ctl[AP_CTL_SIZE];
  const int a = *action;
  // max priority over the filled ring, read before this push (agent.py:199): kept in pstat by
  // the learn step when the loop has it (a push of the maximum leaves the maximum unchanged)
  double pm = 0.0;
  if (!L.pstat)
    for (int64_t i = tid; i < size; i += blockDim.x) pm = fmax(pm, L.r_prio[i]);
  for (int o = 16; o; o >>= 1) pm = fmax(pm, __shfl_xor_sync(0xffffffffu, pm, o));
  if ((tid & 31) == 0) s_prio[tid >> 5] = pm;
  // the transition's state: the current row, before it changes
  float* rs = L.r_states + slot * L.r_ld;
  for (int j = tid; j <= n; j += blockDim.x) rs[j] = L.state[j];
  // newly decided candidates (envs.py:150-159)
  int np_ = 0, nr_ = 0;
  if (!conflict)
    for (int j = tid; j < n; j += blockDim.x) {
      const int8_t now = L.status[j], prev = L.decided[j];
      np_ += (now == 1 && prev == -1);
      nr_ += (now == 0 && prev == -1);
    }
  const int nP = block_sum(np_, s_red);
  const int nR = block_sum(nr_, s_red);
  const double reward = conflict ? -1.0 : __dadd_rn(__dmul_rn(0.4, (double)nP), __dmul_rn(0.1, (double)nR));
  if (!conflict)
    for (int j = tid; j < L.ld; j += blockDim.x) {
      L.decided[j] = L.status[j];
      L.seeds[j] = L.seeds_try[j];
    }
  __syncthreads();
  // next decision position: first undecided dim in the order (envs.py:207-211)
  int64_t pos = L.ctl[AP_PL_POS];
  if (!conflict) {
    if (complete) {
      pos = -1;
    } else {
      int first = 0x7fffffff;
      for (int k = tid; k < n; k += blockDim.x)
        if (L.decided[L.order[k]] == -1) first = min(first, k);
      first = block_min(first, s_red);
      pos = first == 0x7fffffff ? -1 : L.order[first];
    }
  }
  const bool done = conflict || complete;
  // next state row (envs.py:213-220) -> ring next_states; transition fields
  float* rn = L.r_next + slot * L.r_ld;
  for (int j = tid; j < n; j += blockDim.x) rn[j] = (float)L.decided[j];
  if (tid == 0) {
    rn[n] = position_feature(pos, n);
    L.r_actions[slot] = a;
    L.r_rewards[slot] = (float)reward;
    L.r_done[slot] = done;
    double pmax = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) pmax = fmax(pmax, s_prio[w]);
    if (L.pstat) {
      if (!size) L.pstat[0] = L.pstat[1] = 1.0;  // 1.0 ** alpha == 1.0
      L.r_prio[slot] = L.pstat[0];
      L.r_scaled[slot] = L.pstat[1];
    } else {
      L.r_prio[slot] = size ? pmax : 1.0;
    }
    L.log_reward[step] = reward;
  }
  for (int k = tid; k < L.num_actions; k += blockDim.x) L.r_mask[slot * L.num_actions + k] = done ? 0 : 1;
  // partitions of a completed plan (envs.py:192-194)
  int parts = 0;
  if (complete)
    for (int j = tid; j < n; j += blockDim.x) parts += L.decided[j] == 1;
  parts = block_sum(parts, s_red);
  __shared__ int s_better;
  if (tid == 0) {
    const double total = __dadd_rn(L.dctl[AP_PLD_TOTAL], reward);  // total += result.reward (cli.py:233)
    L.dctl[AP_PLD_TOTAL] = total;
    L.ctl[AP_PL_EP_STEPS] += 1;
    s_better = 0;
    if (done) {
      const int64_t ep = L.ctl[AP_PL_EPISODES];
      L.ep_conflict[ep] = conflict;
      L.ep_len[ep] = (int32_t)L.ctl[AP_PL_EP_STEPS];
      L.ep_return[ep] = total;
      // incumbent: strictly greater (partitions, return), first wins (cli.py:237-240)
      if (!conflict) {
        const int64_t bp = L.ctl[AP_PL_BEST_PART];
        const double br = L.dctl[AP_PLD_BEST_REWARD];
        if (bp < 0 || parts > bp || (parts == bp && total > br)) {
          L.ctl[AP_PL_BEST_PART] = parts;
          L.dctl[AP_PLD_BEST_REWARD] = total;
          L.ctl[AP_PL_BEST_EP] = L.ctl[AP_PL_EP_BASE] + ep;
          s_better = 1;
        }
      }
      L.ctl[AP_PL_EPISODES] = ep + 1;
      L.ctl[AP_PL_EP_STEPS] = 0;
      L.dctl[AP_PLD_TOTAL] = 0.0;
    }
    L.ctl[AP_PL_STEP] = step + 1;
    L.ctl[AP_PL_GEN] += 1;
    L.ctl[AP_PL_SYNC] = 0;  // raised by this step's learn tail when a target sync is due
    L.ctl[AP_CTL_SLOT] = (slot + 1) % L.cap;
    L.ctl[AP_CTL_SIZE] = size + 1 < L.cap ? size + 1 : L.cap;
  }
  __syncthreads();
  if (s_better)
    for (int j = tid; j < L.ld; j += blockDim.x) L.best_row[j] = L.decided[j];
  __syncthreads();
  // the env for the next step: reset to the template after a finished episode
  if (done) {
    for (int j = tid; j < L.ld; j += blockDim.x) {
      L.seeds[j] = L.t_seeds[j];
      L.decided[j] = L.t_decided[j];
    }
    if (tid == 0) L.ctl[AP_PL_POS] = L.ctl[AP_PL_T_POS];
    __syncthreads();
    for (int j = tid; j < n; j += blockDim.x) L.state[j] = (float)L.decided[j];
    if (tid == 0) L.state[n] = position_feature(L.ctl[AP_PL_T_POS], n);
  } else {
    for (int j = tid; j < n; j += blockDim.x) L.state[j] = (float)L.decided[j];
    if (tid == 0) {
      L.state[n] = position_feature(pos, n);
      L.ctl[AP_PL_POS] = pos;
    }
  }
}

// B random() draws for rng.choice's uniforms (agent.py:220)
__device__ __forceinline__ bool learn_gated_off(const ap_parity_loop& L) {
  return L.learn_gate > 0 && L.ctl[AP_CTL_SIZE] < L.learn_gate;
}

// agent.learn's draws and PER sample in one CTA: B random() draws (rng.choice's uniforms,
// agent.py:220), each thread jumping the PCG64 stream ahead to its own draw, then the PER
// sample (per_sample.cuh) with the priorities and cdf staged in shared memory when they fit.
// Early mode (see ap_parity_sample): the ring and stream as the step starts, the act's draws
// replayed, the pending push counted, the read acknowledged, the final stream in rng_next.
constexpr int kSampleThreads = 512;  // (128 registers per thread: the cumsum keeps 32 operands in flight)

// PCG64 jump-ahead by k <= kSampleMaxB steps without the square-and-multiply loop:
// state_k = M^k state_0 + S_k inc with S_k = 1 + M + ... + M^(k-1) (mod 2^128), both tabulated at
// compile time (w[k] = {M^k hi, lo, S_k hi, lo}).
struct JumpTable {
  uint64_t w[kSampleMaxB + 1][4];
};
constexpr JumpTable make_jump_table() {
  JumpTable t{};
  const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;  // pcg_mult()
  u128 m = 1, sum = 0;
  for (int k = 0; k <= kSampleMaxB; ++k) {
    t.w[k][0] = (uint64_t)(m >> 64), t.w[k][1] = (uint64_t)m;
    t.w[k][2] = (uint64_t)(sum >> 64), t.w[k][3] = (uint64_t)sum;
    sum = sum * mult + 1;
    m = m * mult;
  }
  return t;
}
__constant__ JumpTable g_jump = make_jump_table();

__device__ __forceinline__ u128 pcg_jump(u128 state, u128 inc, int k) {
  const u128 m = ((u128)g_jump.w[k][0] << 64) | (u128)g_jump.w[k][1];
  const u128 sum = ((u128)g_jump.w[k][2] << 64) | (u128)g_jump.w[k][3];
  return m * state + sum * inc;
}

constexpr int kSampleSmemBytes = 190 * 1024;  // + ~30 KB static <= 227 KB

__global__ void __launch_bounds__(kSampleThreads) parity_sample_kernel(ap_parity_loop L, int B, double alpha,
                                                                       double beta, double* scratch, int32_t* idx,
                                                                       float* w, double* u_out, uint64_t* rng_next,
                                                                       int early, int smem_doubles) {
  pdl_entry();
  extern __shared__ double dyn[];
  __shared__ PerShared S;
  __shared__ double su[kSampleMaxB];
  __shared__ uint64_t s_rng[6];
  const int tid = threadIdx.x, nt = blockDim.x;
  ST(0);
  // every thread reads the control words it needs, then a barrier: in early mode nothing is
  // read from the control block after the acknowledgement (env.step advances slot / size)
  const int64_t* c = L.ctl;
  bool go;
  int64_t slot, size;
  if (early) {
    go = c[AP_PL_EPISODES] < c[AP_PL_BUDGET] && c[AP_PL_STEP] < c[AP_PL_MAX_STEPS];
    slot = c[AP_CTL_SLOT];
    size = c[AP_CTL_SIZE];
  } else {
    go = c[AP_PL_ACTIVE] != 0;
    slot = -1;
    size = c[AP_CTL_SIZE] - 1;  // the ring before this step's push (n below is the pushed size)
  }
  const int n = (int)(size + 1 < L.cap ? size + 1 : L.cap);
  const int64_t gen = early ? c[AP_PL_GEN] : 0, train = early ? c[AP_CTL_TRAIN] : 0;
  const bool active = go;  // the step runs (the act waits for this kernel's acknowledgement)
  go = go && !(L.learn_gate > 0 && n < L.learn_gate) && n >= B;
  __syncthreads();
  if (tid == 0) {
    NpPcg64 g = NpPcg64::load(L.rng);
    if (early && go) {
      // the act's draws (agent.py:161-166): they depend on the step count, not on Q
      const double eps = epsilon_at(train, L.eps_start, L.eps_final, L.eps_decay);
      if (g.next_double() < eps) (void)g.integers(L.num_actions);
    }
    g.store(s_rng);
    // every read of the stream / control block is done: the act may advance the stream
    if (early && active)
      asm volatile("st.release.gpu.u64 [%0], %1;" ::"l"(L.ctl + AP_PL_ACK), "l"(gen + 1) : "memory");
  }
  if (!go) return;
  const bool staged = 2 * (int64_t)n + B <= smem_doubles;
  if (tid == 32) per_tree(n, S);
  // scaled = priorities ** alpha: early mode from the cache (+ the pending push: the ring's max
  // priority and its power, kept by env.step / the learn step), late mode computed
  const double sub = early ? L.pstat[1] : 0.0;
  for (int i = tid; i < n; i += nt) {
    const double v = early ? (i == slot ? sub : __ldcg(L.r_scaled + i)) : pow(L.r_prio[i], alpha);
    if (staged)
      dyn[i] = v;
    else
      scratch[i] = v;
  }
  __syncthreads();
  ST(1);
  // (two inlined copies: with the shared-memory arrays the compiler knows their space)
  if (staged) {
    per_total(dyn, S);
    ST(2);
    per_cdf(dyn, n, dyn + n, S);
  } else {
    per_total(scratch, S);
    ST(2);
    per_cdf(scratch, n, scratch + L.cap, S);
  }
  // the B uniforms, by the threads the cdf chain leaves idle
  const u128 s0 = ((u128)s_rng[0] << 64) | (u128)s_rng[1], inc = ((u128)s_rng[2] << 64) | (u128)s_rng[3];
  for (int b = nt - 1 - tid; tid != 0 && b < B; b += nt - 1) {
    u128 st = pcg_jump(s0, inc, b);
    const double v = pcg_next_double(st, inc);  // draw b: the state after b + 1 steps
    su[b] = v;
    if (u_out) u_out[b] = v;
    if (b == B - 1) {  // random() leaves the 32-bit buffer alone
      uint64_t* dst = early ? rng_next : L.rng;
      dst[0] = (uint64_t)(st >> 64);
      dst[1] = (uint64_t)st;
      if (early) dst[2] = s_rng[2], dst[3] = s_rng[3], dst[4] = s_rng[4], dst[5] = s_rng[5];
    }
  }
  __syncthreads();
  if (staged)
    per_pick(dyn, n, beta, su, B, dyn + n, idx, w, S);
  else
    per_pick(scratch, n, beta, su, B, scratch + L.cap, idx, w, S);
  ST(3);
}

__global__ void per_scaled_kernel(const double* __restrict__ prio, int64_t n, double alpha, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = pow(prio[i], alpha);
}

// pstat = {max priority over the ring (1.0 when empty), its ** alpha}: one CTA
__global__ void per_pstat_kernel(const double* __restrict__ prio, int64_t n, double alpha, double* __restrict__ pstat) {
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, prio[i]);
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) m = fmax(m, red[k]);
    m = fmax(m, red[0]);
    pstat[0] = n ? m : 1.0;
    pstat[1] = pow(pstat[0], alpha);
  }
}

// loss log, train-step counter, target-sync flag (agent.py:325-337)
__global__ void parity_learn_tail_kernel(ap_parity_loop L, const float* __restrict__ loss, int sync_every) {
  pdl_entry();
  if (threadIdx.x || learn_gated_off(L)) return;
  const int64_t t = L.ctl[AP_CTL_TRAIN];
  const int64_t k = t - L.ctl[AP_PL_TRAIN0];
  const float v = *loss;
  if (k >= 0 && k < L.loss_cap) L.loss_log[k] = v;
  if (!isfinite(v) && L.ctl[AP_PL_LOSS_BAD] < 0) L.ctl[AP_PL_LOSS_BAD] = k;
  L.ctl[AP_CTL_TRAIN] = t + 1;
  L.ctl[AP_PL_SYNC] = ((t + 1) % sync_every) == 0;
}

struct SyncSegs {
  const float* src[8];
  float* dst[8];
  int64_t count[8];
  int n;
};

// hard target sync (agent.py:142-144) when the learn tail raised the flag
__global__ void parity_sync_kernel(const int64_t* __restrict__ ctl, SyncSegs s) {
  pdl_entry();
  if (!ctl[AP_PL_SYNC]) return;
  for (int k = 0; k < s.n; ++k)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < s.count[k];
         i += (int64_t)gridDim.x * blockDim.x)
      s.dst[k][i] = s.src[k][i];
}

__global__ void loop_learn_cond_kernel(cudaGraphConditionalHandle h, const int64_t* ctl, int64_t batch) {
  cudaGraphSetConditional(h, ctl[AP_CTL_SIZE] >= batch ? 1u : 0u);
}

__global__ void loop_continue_cond_kernel(cudaGraphConditionalHandle h, const int64_t* ctl) {
  cudaGraphSetConditional(h, (ctl[AP_PL_EPISODES] < ctl[AP_PL_BUDGET] && ctl[AP_PL_STEP] < ctl[AP_PL_MAX_STEPS]) ? 1u
                                                                                                            : 0u);
}

}  // namespace
}  // namespace apb

struct ap_loop {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

using namespace apb;

extern "C" {

int ap_parity_act(const ap_parity_loop* L, const float* q, int32_t* action, void* stream) {
  if (!L || !q || !action || !L->ctl || !L->rng) {
    set_error("ap_parity_act: null argument");
    return AP_ERR_INVALID;
  }
  launch_pdl(parity_act_kernel, dim3(1), dim3(kPostThreads), 0, (cudaStream_t)stream, *L, q, action);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_parity_post(const ap_parity_loop* L, const int32_t* action, void* stream) {
  if (!L || !action || L->n < 1 || L->cap < 1) {
    set_error("ap_parity_post: bad arguments");
    return AP_ERR_INVALID;
  }
  launch_pdl(parity_post_kernel, dim3(1), dim3(kPostThreads), 0, (cudaStream_t)stream, *L, action);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_parity_sample(const ap_parity_loop* L, int32_t B, double alpha, double beta, double* scratch,
                     int32_t* indices, float* weights, double* uniforms_out, uint64_t* rng_next, int32_t early,
                     void* stream) {
  if (!L || !L->ctl || !L->rng || !L->r_prio || !scratch || !indices || !weights || B < 1 || B > kSampleMaxB ||
      (early && !rng_next)) {
    set_error("ap_parity_sample: bad arguments (1 <= B <= 1024; early mode needs rng_next)");
    return AP_ERR_INVALID;
  }
  static PerDeviceMax configured;
  const int64_t want = (2 * L->cap + B) * (int64_t)sizeof(double);
  const int smem = want <= kSampleSmemBytes ? (int)want : 0;
  if (smem && configured.need(current_device(), smem))
    AP_CUDA_CHECK(cudaFuncSetAttribute(parity_sample_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  launch_pdl(parity_sample_kernel, dim3(1), dim3(kSampleThreads), (size_t)smem, (cudaStream_t)stream, *L, (int)B,
             alpha, beta, scratch, indices, weights, uniforms_out, rng_next, (int)(early != 0),
             smem / (int)sizeof(double));
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_per_scaled(const double* priorities, int64_t n, double alpha, double* scaled, double* pstat, void* stream) {
  if (n < 0 || (n && (!priorities || !scaled))) {
    set_error("ap_per_scaled: bad arguments");
    return AP_ERR_INVALID;
  }
  if (pstat) per_pstat_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(priorities, n, alpha, pstat);
  if (!n) return AP_OK;
  per_scaled_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, (cudaStream_t)stream>>>(priorities, n,
                                                                                                   alpha, scaled);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_parity_learn_tail(const ap_parity_loop* L, const float* loss, int32_t sync_every, void* stream) {
  if (!L || !loss || sync_every < 1) {
    set_error("ap_parity_learn_tail: bad arguments");
    return AP_ERR_INVALID;
  }
  launch_pdl(parity_learn_tail_kernel, dim3(1), dim3(32), 0, (cudaStream_t)stream, *L, loss, (int)sync_every);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_parity_target_sync(const int64_t* ctl, int32_t n, const float* const* src, float* const* dst,
                          const int64_t* count, void* stream) {
  if (!ctl || n < 0 || n > 8) {
    set_error("ap_parity_target_sync: at most 8 segments");
    return AP_ERR_INVALID;
  }
  SyncSegs s = {};
  s.n = n;
  int64_t most = 0;
  for (int k = 0; k < n; ++k) {
    s.src[k] = src[k];
    s.dst[k] = dst[k];
    s.count[k] = count[k];
    most = std::max<int64_t>(most, count[k]);
  }
  const int blocks = (int)std::min<int64_t>(std::max<int64_t>((most + 255) / 256, 1), 296);
  launch_pdl(parity_sync_kernel, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, ctl, s);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_pcg64_host_draws(uint64_t* state6, const int64_t* ops, int32_t n, double* out) {
  if (!state6 || (n > 0 && (!ops || !out))) {
    set_error("ap_pcg64_host_draws: null argument");
    return AP_ERR_INVALID;
  }
  NpPcg64 g = NpPcg64::load(state6);
  for (int32_t i = 0; i < n; ++i) {
    if (ops[i] < 1 || ops[i] > (int64_t(1) << 32)) {
      if (ops[i] == 0) {
        out[i] = g.next_double();
        continue;
      }
      set_error("ap_pcg64_host_draws: op must be 0 (random) or 1..2^32 (integers(op))");
      return AP_ERR_INVALID;
    }
    out[i] = (double)g.integers(ops[i]);
  }
  g.store(state6);
  return AP_OK;
}

int ap_loop_graph_create(void* step_graph, void* learn_graph, const int64_t* ctl, int64_t batch, ap_loop_t* out) {
  if (!step_graph || !ctl || !out || batch < 1) {
    set_error("ap_loop_graph_create: bad arguments");
    return AP_ERR_INVALID;
  }
  ap_loop* lp = new (std::nothrow) ap_loop();
  if (!lp) {
    set_error("ap_loop_graph_create: out of host memory");
    return AP_ERR_INVALID;
  }
  auto fail = [&](cudaError_t e, const char* what) {
    if (lp->graph) cudaGraphDestroy(lp->graph);
    delete lp;
    return cuda_fail(e, what);
  };
  cudaError_t e;
  if ((e = cudaGraphCreate(&lp->graph, 0)) != cudaSuccess) return fail(e, "cudaGraphCreate");
  cudaGraphConditionalHandle h_loop, h_learn;
  if ((e = cudaGraphConditionalHandleCreate(&h_loop, lp->graph, 1, cudaGraphCondAssignDefault)) != cudaSuccess)
    return fail(e, "cudaGraphConditionalHandleCreate(loop)");
  if (learn_graph &&
      (e = cudaGraphConditionalHandleCreate(&h_learn, lp->graph, 0, cudaGraphCondAssignDefault)) != cudaSuccess)
    return fail(e, "cudaGraphConditionalHandleCreate(learn)");
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = h_loop;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  if ((e = cudaGraphAddNode(&wnode, lp->graph, nullptr, 0, &wp)) != cudaSuccess) return fail(e, "add WHILE node");
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  cudaGraphNode_t n_step, n_lcond, n_if, n_cont;
  if ((e = cudaGraphAddChildGraphNode(&n_step, body, nullptr, 0, (cudaGraph_t)step_graph)) != cudaSuccess)
    return fail(e, "add step child graph");
  n_if = n_step;  // no learn graph: the step graph holds a self-gated learn body (learn_gate)
  if (learn_graph) {
    {
      cudaKernelNodeParams kp = {};
      int64_t b = batch;
      void* args[] = {&h_learn, (void*)&ctl, &b};
      kp.func = (void*)loop_learn_cond_kernel;
      kp.gridDim = dim3(1);
      kp.blockDim = dim3(1);
      kp.kernelParams = args;
      if ((e = cudaGraphAddKernelNode(&n_lcond, body, &n_step, 1, &kp)) != cudaSuccess)
        return fail(e, "add learn-condition kernel");
    }
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = h_learn;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    if ((e = cudaGraphAddNode(&n_if, body, &n_lcond, 1, &ip)) != cudaSuccess) return fail(e, "add IF node");
    cudaGraphNode_t n_learn;
    if ((e = cudaGraphAddChildGraphNode(&n_learn, ip.conditional.phGraph_out[0], nullptr, 0,
                                        (cudaGraph_t)learn_graph)) != cudaSuccess)
      return fail(e, "add learn child graph");
  }
  {
    cudaKernelNodeParams kp = {};
    void* args[] = {&h_loop, (void*)&ctl};
    kp.func = (void*)loop_continue_cond_kernel;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = args;
    if ((e = cudaGraphAddKernelNode(&n_cont, body, &n_if, 1, &kp)) != cudaSuccess)
      return fail(e, "add loop-condition kernel");
  }
  if ((e = cudaGraphInstantiate(&lp->exec, lp->graph, 0)) != cudaSuccess) return fail(e, "cudaGraphInstantiate");
  *out = lp;
  return AP_OK;
}

int ap_loop_graph_launch(ap_loop_t lp, void* stream) {
  if (!lp || !lp->exec) {
    set_error("ap_loop_graph_launch: null loop");
    return AP_ERR_INVALID;
  }
  AP_CUDA_CHECK(cudaGraphLaunch(lp->exec, (cudaStream_t)stream));
  return AP_OK;
}

int ap_loop_graph_destroy(ap_loop_t lp) {
  if (!lp) return AP_OK;
  if (lp->exec) cudaGraphExecDestroy(lp->exec);
  if (lp->graph) cudaGraphDestroy(lp->graph);
  delete lp;
  return AP_OK;
}

}  // extern "C"
