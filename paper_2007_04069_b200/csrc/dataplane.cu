// PP-infer data plane on the device: batched synthetic
// profiles, bit-identical to the reference's generate_environment for the
// uniform distribution (reference dataproc.py:123-145, build_environment_arrays
// dataproc.py:99-120, coarsen dataproc.py:79-96).
//
// numpy's default_rng(seed) is PCG64 (XSL-RR 128/64): each draw advances the
// 128-bit LCG state = state * M + inc and outputs rotr64(hi ^ lo, state >> 122)
// of the new state; Generator.uniform(0, 1) is (x >> 11) * 2^-53.  The host
// passes each environment's initial (state, inc) as numpy computes them from
// the seed (SeedSequence); the device reproduces the stream.  The three draws
// c, a, w are stream positions [0, n), [n, 2n), [2n, 3n): every thread jumps
// ahead (PCG's O(log k) advance) to its slice and steps sequentially.
// Then, as the reference: naive sequential cumsum of c and w, right-endpoint
// coarsening to G points, joint scaling by max(cs, as, ws, 0).
//
// normal / binomial profiles use numpy's ziggurat / BTPE rejection samplers
// (np_samplers.cuh), which consume a data-dependent number of draws: one thread
// walks one environment's stream sequentially, keeping the running cumsums and
// capturing the coarse points as their source index passes.
#include <algorithm>
#include <cstdint>

#include "engine.h"
#include "pcg64.cuh"
#include "np_samplers.cuh"

namespace apb {
namespace {

constexpr int kGenThreads = 256;

__global__ void __launch_bounds__(kGenThreads) uniform_env_kernel(const uint64_t* seeds4, int64_t E, int n, int G,
                                                                 double* out) {
  extern __shared__ double s_draw[];  // [3n]: c, a, w
  __shared__ double s_max[kGenThreads / 32];
  for (int64_t e = blockIdx.x; e < E; e += gridDim.x) {
    const uint64_t* q = seeds4 + 4 * e;
    const u128 state0 = ((u128)q[0] << 64) | (u128)q[1];
    const u128 inc = ((u128)q[2] << 64) | (u128)q[3];
    const int total = 3 * n;
    const int chunk = (total + kGenThreads - 1) / kGenThreads;
    const int lo = threadIdx.x * chunk, hi = min(total, lo + chunk);
    if (lo < hi) {
      u128 st = pcg_advance(state0, inc, (uint64_t)lo);
      for (int k = lo; k < hi; ++k) s_draw[k] = pcg_next_double(st, inc);
    }
    __syncthreads();
    // np.cumsum (sequential) of c and w, one thread each
    if (threadIdx.x < 2) {
      double* x = s_draw + (threadIdx.x == 0 ? 0 : 2 * n);
      double acc = x[0];
      for (int i = 1; i < n; ++i) {
        acc = acc + x[i];
        x[i] = acc;
      }
    }
    __syncthreads();
    // coarsen (right endpoints; arrays shorter than G are padded with their last value)
    double m = 0.0;
    double* o = out + e * 3 * (int64_t)G;
    for (int i = threadIdx.x; i < G; i += kGenThreads) {
      const int src = n >= G ? (int)(((int64_t)(i + 1) * n) / G - 1) : min(i, n - 1);
      const double c = s_draw[src], a = s_draw[n + src], w = s_draw[2 * n + src];
      o[i] = c;
      o[G + i] = a;
      o[2 * G + i] = w;
      m = fmax(m, fmax(c, fmax(a, w)));
    }
    for (int off = 16; off; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = m;
    __syncthreads();
    double peak = 0.0;
    for (int k = 0; k < kGenThreads / 32; ++k) peak = fmax(peak, s_max[k]);
    if (peak > 0.0)
      for (int i = threadIdx.x; i < 3 * G; i += kGenThreads) o[i] = o[i] / peak;
    __syncthreads();  // s_draw / s_max reused by the next environment
  }
}

// generate_environment(normal | binomial, n, seed) (dataproc.py:123-145), one thread
// per environment: c, a, w drawn in the reference's order (n each), c and w as the
// naive cumsum, right-endpoint coarsening to G points, joint scaling by the maximum.
// kind 1: clip(0.5 + 0.15 * z, 0, 1); kind 2: binomial(100, 0.5) / 100.
__host__ __device__ inline void sampled_env(const uint64_t* q, int n, int G, int kind, double* o) {
  NpPcg64 g;
  g.state = ((u128)q[0] << 64) | (u128)q[1];
  g.inc = ((u128)q[2] << 64) | (u128)q[3];
  g.has_uint32 = 0;
  g.uinteger = 0;
  double peak = 0.0;
  for (int arr = 0; arr < 3; ++arr) {
    const bool prefix = arr != 1;  // C and W are prefix sums, A stays pointwise
    double acc = 0.0;
    int j = 0;  // next coarse point
    for (int i = 0; i < n; ++i) {
      double x;
      if (kind == 1) {
        x = 0.5 + 0.15 * np_standard_normal(g);  // -fmad=false: product and sum rounded separately
        x = fmin(fmax(x, 0.0), 1.0);              // np.clip(.., 0.0, 1.0)
      } else {
        x = (double)np_binomial(g, 100, 0.5) / 100.0;
      }
      acc = (prefix && i > 0) ? acc + x : x;
      if (n >= G) {
        // right endpoint of coarse point j: floor((j + 1) * n / G) - 1
        while (j < G && ((int64_t)(j + 1) * n) / G - 1 == i) {
          o[arr * G + j] = acc;
          peak = fmax(peak, acc);
          ++j;
        }
      } else if (j == i) {  // shorter inputs: point j takes source j
        o[arr * G + j] = acc;
        peak = fmax(peak, acc);
        ++j;
      }
    }
    for (; j < G; ++j) {  // n < G: right padding with the last value
      o[arr * G + j] = acc;
      peak = fmax(peak, acc);
    }
  }
  if (peak > 0.0)
    for (int i = 0; i < 3 * G; ++i) o[i] = o[i] / peak;
}

__global__ void __launch_bounds__(128) sampled_env_kernel(const uint64_t* __restrict__ seeds4, int64_t E, int n, int G,
                                                         int kind, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  sampled_env(seeds4 + 4 * e, n, G, kind, out + e * 3 * (int64_t)G);
}

// Slot statuses for host consumers: K1's int8 slot rows (-1 undecided, 0 R,
// 1 P; sharding.py:36-48 DimStatus) packed 2 bits per slot, code = status + 1,
// slot j of a row in bits 2*(j%4) of byte j/4.  One thread packs one 16-byte
// chunk (16 slots) into one 32-bit word: 16-byte loads and 4-byte stores, both
// coalesced along the row; codes past n are 0, so padding never leaks.
__global__ void __launch_bounds__(256) pack_slots2_kernel(const int8_t* __restrict__ slots, int64_t batch,
                                                          int64_t ld, int64_t n, uint8_t* __restrict__ out,
                                                          int64_t out_ld) {
  const int64_t chunks = (n + 15) / 16, total = batch * chunks;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / chunks, c = t - r * chunks, j0 = c * 16;
    const int4 v = __ldcs(reinterpret_cast<const int4*>(slots + r * ld + j0));
    const uint32_t w[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
    uint32_t packed = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const uint32_t code = ((w[k >> 2] >> (8 * (k & 3))) + 1u) & 3u;  // -1 -> 0, 0 -> 1, 1 -> 2
      packed |= (j0 + k < n ? code : 0u) << (2 * k);
    }
    *reinterpret_cast<uint32_t*>(out + r * out_ld + c * 4) = packed;
  }
}

}  // namespace
}  // namespace apb

using namespace apb;

extern "C" {

int ap_generate_uniform_envs(const uint64_t* pcg_states, int64_t num_envs, int32_t n, int32_t granularity,
                             double* arrays_out, void* stream) {
  if (num_envs < 0 || n < 1 || granularity < 1 || (num_envs > 0 && (!pcg_states || !arrays_out))) {
    set_error("ap_generate_uniform_envs: bad arguments");
    return AP_ERR_INVALID;
  }
  const size_t smem = (size_t)3 * n * sizeof(double);
  if (smem > 200 * 1024) {
    set_error("ap_generate_uniform_envs: n > 8533 does not fit the shared-memory draw buffer");
    return AP_ERR_UNSUPPORTED;
  }
  if (num_envs == 0) return AP_OK;
  AP_CUDA_CHECK(cudaFuncSetAttribute(uniform_env_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  AP_CUDA_CHECK(cudaGetDevice(&dev));
  AP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t grid = std::min<int64_t>(num_envs, (int64_t)sms * 8);
  uniform_env_kernel<<<(unsigned)grid, kGenThreads, smem, (cudaStream_t)stream>>>(pcg_states, num_envs, n, granularity,
                                                                                  arrays_out);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_generate_envs(int32_t kind, const uint64_t* pcg_states, int64_t num_envs, int32_t n, int32_t granularity,
                     double* arrays_out, void* stream) {
  if (kind == 0) return ap_generate_uniform_envs(pcg_states, num_envs, n, granularity, arrays_out, stream);
  if ((kind != 1 && kind != 2) || num_envs < 0 || n < 1 || granularity < 1 ||
      (num_envs > 0 && (!pcg_states || !arrays_out))) {
    set_error("ap_generate_envs: bad arguments (kind 0 uniform, 1 normal, 2 binomial)");
    return AP_ERR_INVALID;
  }
  if (num_envs == 0) return AP_OK;
  const int64_t grid = (num_envs + 127) / 128;
  sampled_env_kernel<<<(unsigned)grid, 128, 0, (cudaStream_t)stream>>>(pcg_states, num_envs, n, granularity, kind,
                                                                        arrays_out);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_generate_envs_host(int32_t kind, const uint64_t* pcg_states, int64_t num_envs, int32_t n,
                          int32_t granularity, double* arrays_out) {
  if ((kind != 1 && kind != 2) || num_envs < 0 || n < 1 || granularity < 1 ||
      (num_envs > 0 && (!pcg_states || !arrays_out))) {
    set_error("ap_generate_envs_host: bad arguments (kind 1 normal, 2 binomial)");
    return AP_ERR_INVALID;
  }
  for (int64_t e = 0; e < num_envs; ++e)
    sampled_env(pcg_states + 4 * e, n, granularity, kind, arrays_out + e * 3 * (int64_t)granularity);
  return AP_OK;
}

int ap_np_samples_host(uint64_t* state6, int32_t kind, int64_t count, int64_t bin_n, double bin_p, double* out) {
  if (!state6 || count < 0 || (count > 0 && !out) || (kind != 0 && kind != 1)) {
    set_error("ap_np_samples_host: bad arguments (kind 0 standard_normal, 1 binomial)");
    return AP_ERR_INVALID;
  }
  NpPcg64 g = NpPcg64::load(state6);
  for (int64_t i = 0; i < count; ++i) out[i] = kind == 0 ? np_standard_normal(g) : (double)np_binomial(g, bin_n, bin_p);
  g.store(state6);
  return AP_OK;
}

int ap_pack_slots2(const int8_t* slots_dev, int64_t batch, int64_t slots_stride, int64_t num_slots, uint8_t* packed_dev,
                   int64_t packed_stride, void* stream) {
  const int64_t need = ((num_slots + 15) / 16) * 4;
  if (batch < 0 || num_slots < 0 || slots_stride < ((num_slots + 15) / 16) * 16 || slots_stride % 16 ||
      packed_stride < need || packed_stride % 4 || (batch > 0 && (!slots_dev || !packed_dev)) ||
      ((uintptr_t)slots_dev % 16) || ((uintptr_t)packed_dev % 4)) {
    set_error("ap_pack_slots2: bad arguments (slot rows 16-byte aligned and padded, packed rows >= 4*ceil(n/16) bytes)");
    return AP_ERR_INVALID;
  }
  if (batch == 0 || num_slots == 0) return AP_OK;
  int dev = 0, sms = 148;
  AP_CUDA_CHECK(cudaGetDevice(&dev));
  AP_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t total = batch * ((num_slots + 15) / 16);
  // oversubscribed grid (8 resident 256-thread CTAs per SM, 64 waves' worth): fewer grid-stride trips
  const int64_t grid = std::min<int64_t>((total + 255) / 256, (int64_t)sms * 64);
  pack_slots2_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(slots_dev, batch, slots_stride, num_slots,
                                                                       packed_dev, packed_stride);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

}  // extern "C"
