// Fused data-parallel step for the DQN learners: Q-gradient all-reduce over
// NVLink peer memory + Adam, one kernel, no NCCL call.
//
// Each rank owns a symmetric exchange buffer xbuf[2][n] (torch symmetric
// memory: every rank can load every peer's buffer over NVLink) and a flag row
// pad[W].  For learn step t (epoch e = ctl[AP_CTL_TRAIN] + 1):
//   1. every CTA copies its slice of the local gradient into xbuf[e & 1];
//   2. the last CTA to finish (device-scope counter) publishes e into every
//      peer's pad[rank] with a system-scope release store; every CTA then
//      acquire-spins on its own pad until all W slots reached e;
//   3. each element is averaged over the W ranks' xbuf[e & 1] in rank order
//      (identical bits on every rank, so the replicas stay identical) and the
//      Adam update is applied to the local parameters.
// Reuse of xbuf[e & 1] at step t + 2 is safe: its copy runs after the step
// t + 1 barrier, which every peer reaches only after finishing step t.  The
// grid is at most one CTA per SM so all CTAs are co-resident while spinning.
#include <algorithm>

#include "engine.h"

namespace apb {
namespace {

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kMaxWorld = 8;

struct DpArgs {
  const float* grad;
  float* xbuf[kMaxWorld];   // peers' exchange buffers [2][n]
  uint32_t* pad[kMaxWorld];  // peers' flag rows [W]
  int world, rank;
  int64_t n;
  float* params;
  float* m;
  float* v;
  float lr, b1, b2, eps;
  const int64_t* ctl;
  unsigned int* counter;  // local, zero between calls
};

__global__ void __launch_bounds__(256) dp_allreduce_adam_kernel(DpArgs a) {
  const uint32_t epoch = (uint32_t)(a.ctl[AP_CTL_TRAIN] + 1);
  const int64_t half = (int64_t)(epoch & 1u) * a.n;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  // 1. publish the local gradient
  float* mine = a.xbuf[a.rank] + half;
  for (int64_t i = tid; i < a.n; i += nt) mine[i] = a.grad[i];
  __threadfence_system();
  __syncthreads();
  // 2. cross-rank barrier
  __shared__ float s_c[2];
  if (threadIdx.x == 0) {
    if (atomicAdd(a.counter, 1u) == gridDim.x - 1) {
      *a.counter = 0;
      for (int p = 0; p < a.world; ++p) st_release_sys(a.pad[p] + a.rank, epoch);
    }
    const uint32_t* own = a.pad[a.rank];
    for (int p = 0; p < a.world; ++p)
      while ((int32_t)(ld_acquire_sys(own + p) - epoch) < 0) {
      }
    const double t = (double)epoch;  // Adam step (agent.py:240-250)
    s_c[0] = (float)(1.0 - pow((double)a.b1, t));
    s_c[1] = (float)(1.0 - pow((double)a.b2, t));
  }
  __syncthreads();
  const float c1 = s_c[0], c2 = s_c[1], inv = 1.0f / (float)a.world;
  // 3. average in rank order + Adam
  for (int64_t i = tid; i < a.n; i += nt) {
    float g = 0.0f;
    for (int p = 0; p < a.world; ++p) g += __ldcg(a.xbuf[p] + half + i);
    g *= inv;
    const float mi = a.b1 * a.m[i] + (1.0f - a.b1) * g;
    const float vi = a.b2 * a.v[i] + (1.0f - a.b2) * g * g;
    a.m[i] = mi;
    a.v[i] = vi;
    a.params[i] -= a.lr * (mi / c1) / (sqrtf(vi / c2) + a.eps);
  }
}

}  // namespace
}  // namespace apb

using namespace apb;

extern "C" {

int ap_dp_allreduce_adam(int32_t world, int32_t rank, const float* grad, float* const* xbuf_peers,
                         uint32_t* const* pad_peers, int64_t n, float* params, float* m, float* v, float lr,
                         float beta1, float beta2, float eps, const int64_t* ctl, uint32_t* counter, void* stream) {
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world || !grad || !xbuf_peers || !pad_peers ||
      !params || !m || !v || !ctl || !counter || n < 0) {
    set_error("ap_dp_allreduce_adam: bad arguments (world <= 8, host arrays of peer pointers)");
    return AP_ERR_INVALID;
  }
  DpArgs a{};
  a.grad = grad;
  for (int p = 0; p < world; ++p) {
    a.xbuf[p] = xbuf_peers[p];
    a.pad[p] = pad_peers[p];
  }
  a.world = world;
  a.rank = rank;
  a.n = n;
  a.params = params;
  a.m = m;
  a.v = v;
  a.lr = lr;
  a.b1 = beta1;
  a.b2 = beta2;
  a.eps = eps;
  a.ctl = ctl;
  a.counter = reinterpret_cast<unsigned int*>(counter);
  int dev = 0, sms = 0;
  AP_CUDA_CHECK(cudaGetDevice(&dev));
  AP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // co-resident grid (spin barrier): at most one 256-thread CTA per SM
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, (n + 255) / 256));
  dp_allreduce_adam_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

}  // extern "C"
