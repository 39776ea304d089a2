// agent.act of the parity loop (agent.py:155-170) as device functions shared by the
// stand-alone act kernel (parity.cu) and the fused act forward (fused_mlp.cu):
// epsilon-greedy with numpy's draws -- random(), then integers(#actions) when exploring --
// else the first maximum of Q; the K1 input row seeds_try = seeds + this step's decision.
#pragma once

#include <cmath>
#include <cstdint>

#include "engine.h"
#include "pcg64.cuh"

namespace apb {
namespace {  // internal linkage: included by several translation units

__device__ __forceinline__ double epsilon_at(int64_t it, double start, double final_eps, int64_t decay) {
  // agent.py:50-55: start + (final - start) * min(1, max(0, it / decay)), every op rounded
  if (decay <= 0) return final_eps;
  double frac = __ddiv_rn((double)it, (double)decay);
  frac = fmin(1.0, fmax(0.0, frac));
  return __dadd_rn(start, __dmul_rn(__dsub_rn(final_eps, start), frac));
}

// Start of a step: is the loop still running (episodes < budget, log not full)?  With `check`
// off the caller's loop condition already guarantees it.  Thread 0 of one CTA (`writer`)
// records the answer for the step's later kernels.
__device__ __forceinline__ bool parity_step_begin(const ap_parity_loop& L, bool check, bool writer) {
  const bool active =
      !check || (L.ctl[AP_PL_EPISODES] < L.ctl[AP_PL_BUDGET] && L.ctl[AP_PL_STEP] < L.ctl[AP_PL_MAX_STEPS]);
  if (writer) L.ctl[AP_PL_ACTIVE] = active;
  return active;
}

// Early PER sample mode: the step's sampler reads the random stream as the step starts, so the
// act may advance it only after the sampler's acknowledgement (ctl[AP_PL_ACK] == GEN + 1).
// Bounded: a sampler that never ran sets ctl[AP_PL_FAULT] instead of hanging the loop.
__device__ __forceinline__ void parity_wait_sample_ack(const ap_parity_loop& L) {
  if (!L.early_sample) return;
  const int64_t want = L.ctl[AP_PL_GEN] + 1;
  volatile const int64_t* ack = L.ctl + AP_PL_ACK;
  for (int64_t spin = 0; *ack != want; ++spin) {
    if (spin > (1ll << 22)) {  // ~0.3 s
      L.ctl[AP_PL_FAULT] = 1;
      break;
    }
    __nanosleep(64);
  }
  __threadfence();
}

// seeds_try = seeds (and the state-row log) -- every thread of one CTA
__device__ __forceinline__ void parity_act_rows(const ap_parity_loop& L) {
  const int64_t step = L.ctl[AP_PL_STEP];
  for (int j = threadIdx.x; j < L.ld; j += blockDim.x) {
    L.seeds_try[j] = L.seeds[j];
    if (L.log_decided) L.log_decided[step * L.ld + j] = L.decided[j];
  }
}

// the decision itself -- one thread, after parity_act_rows and a CTA barrier
__device__ __forceinline__ void parity_act_decide(const ap_parity_loop& L, const float* q, int32_t* action) {
  const int64_t step = L.ctl[AP_PL_STEP];
  const int64_t pos = L.ctl[AP_PL_POS];
  NpPcg64 g = NpPcg64::load(L.rng);
  const double eps = epsilon_at(L.ctl[AP_CTL_TRAIN], L.eps_start, L.eps_final, L.eps_decay);
  int a;
  if (g.next_double() < eps) {
    // every action is allowed while the episode runs (envs.py:175-179)
    a = (int)g.integers(L.num_actions);
  } else {  // masked argmax, ties to the lowest index (agent.py:147-152)
    a = 0;
    float best = q[0];
    for (int k = 1; k < L.num_actions; ++k)
      if (q[k] > best) best = q[k], a = k;
  }
  parity_wait_sample_ack(L);
  g.store(L.rng);
  *action = a;
  L.seeds_try[pos] = a == 0 ? 1 : 0;  // ACTION_PARTITION seeds P, ACTION_REPLICATE seeds R
  L.log_action[step] = a;
  L.log_pos[step] = (int32_t)pos;
}

}  // namespace
}  // namespace apb
