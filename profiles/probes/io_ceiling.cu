// IO-only ceilings for K1's traffic mix: per plan read round16(D) seed bytes,
// write round16(S) slot bytes + 1 + 16.  Variants:
//   mode 0: warp per plan, st.global.cs        (K1's pattern)
//   mode 1: warp per plan, plain st.global
//   mode 2: warp per plan, prefetched next-plan seeds, st.global.cs
//   mode 3: flat: grid-stride 16-byte copies over the whole seed / slot arrays
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <int MODE>
__device__ __forceinline__ void st16(void* p, uint4 v) {
  if (MODE == 1)
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <int MODE, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) io_kernel(const int8_t* seeds, int64_t ss, int nq_d, int8_t* out,
                                                        int64_t os, int nq_s, uint8_t* outcome, int4* counts,
                                                        int64_t batch) {
  const int lane = threadIdx.x & 31;
  if (MODE == 3) {
    const int64_t n_in = batch * ss / 16, n_out = batch * os / 16;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    uint32_t x = 0;
    for (int64_t i = tid; i < n_in; i += nt) {
      uint4 v = ldg_stream(seeds + 16 * i);
      x ^= v.x ^ v.w;
    }
    for (int64_t i = tid; i < n_out; i += nt) st16<0>(out + 16 * i, make_uint4(x, 1, 2, 3));
    for (int64_t i = tid; i < batch; i += nt) {
      outcome[i] = (uint8_t)x;
      counts[i] = make_int4(x, 1, 2, 3);
    }
    return;
  }
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  int64_t b = blockIdx.x * WARPS + (threadIdx.x >> 5);
  uint4 cur[3];
  if (MODE == 2 && b < batch)
    for (int i = 0; i < 3; ++i) cur[i] = ldg_stream(seeds + b * ss + 16 * min(lane + 32 * i, nq_d - 1));
  for (; b < batch; b += nw) {
    uint32_t x = 0;
    if (MODE == 2) {
      for (int i = 0; i < 3; ++i) x ^= cur[i].x ^ cur[i].w;
      const int64_t bn = b + nw < batch ? b + nw : b;
      for (int i = 0; i < 3; ++i) cur[i] = ldg_stream(seeds + bn * ss + 16 * min(lane + 32 * i, nq_d - 1));
    } else {
      for (int q = lane; q < nq_d; q += 32) {
        uint4 v = ldg_stream(seeds + b * ss + 16 * q);
        x ^= v.x ^ v.y ^ v.z ^ v.w;
      }
    }
    x = __reduce_or_sync(0xffffffffu, x);
    for (int q = lane; q < nq_s; q += 32) st16<MODE>(out + b * os + 16 * q, make_uint4(x, x + 1, x + 2, x + 3));
    if (lane == 0) {
      outcome[b] = (uint8_t)x;
      counts[b] = make_int4(x, 1, 2, 3);
    }
  }
}

template <int MODE, int WARPS>
void run(const char* name, const int8_t* seeds, int nq_d, int8_t* out, int nq_s, uint8_t* oc, int4* cnt, int64_t B,
         int sms, int per_sm) {
  const int D = 1059, S = 5633;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto k = io_kernel<MODE, WARPS>;
  for (int w = 0; w < 3; ++w) k<<<sms * per_sm, WARPS * 32>>>(seeds, nq_d * 16, nq_d, out, nq_s * 16, nq_s, oc, cnt, B);
  cudaEventRecord(e0);
  const int it = 20;
  for (int w = 0; w < it; ++w) k<<<sms * per_sm, WARPS * 32>>>(seeds, nq_d * 16, nq_d, out, nq_s * 16, nq_s, oc, cnt, B);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= it;
  const double alg = (double)(D + S + 17) * B;
  printf("%-28s warps=%2d ctas/sm=%d  %.3f ms  %.1f M plans/s  %.1f GB/s algorithmic\n", name, WARPS, per_sm, ms,
         B / ms / 1e3, alg / ms / 1e6);
}

int main() {
  const int D = 1059, S = 5633;
  const int nq_d = (D + 15) / 16, nq_s = (S + 15) / 16;
  const int64_t B = 1 << 22;
  int8_t *seeds, *out;
  uint8_t* oc;
  int4* cnt;
  cudaMalloc(&seeds, B * nq_d * 16);
  cudaMalloc(&out, B * nq_s * 16);
  cudaMalloc(&oc, B);
  cudaMalloc(&cnt, B * 16);
  cudaMemset(seeds, 1, B * nq_d * 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, 8>("warp/plan .cs", seeds, nq_d, out, nq_s, oc, cnt, B, sms, 4);
  run<1, 8>("warp/plan plain st", seeds, nq_d, out, nq_s, oc, cnt, B, sms, 4);
  run<2, 8>("warp/plan prefetch .cs", seeds, nq_d, out, nq_s, oc, cnt, B, sms, 4);
  run<2, 16>("warp/plan prefetch .cs", seeds, nq_d, out, nq_s, oc, cnt, B, sms, 2);
  run<2, 8>("warp/plan prefetch .cs", seeds, nq_d, out, nq_s, oc, cnt, B, sms, 8);
  run<3, 8>("flat grid-stride", seeds, nq_d, out, nq_s, oc, cnt, B, sms, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int w = 0; w < 10; ++w) cudaMemsetAsync(out, w, B * nq_s * 16);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("memset (write only): %.1f GB/s\n", (double)B * nq_s * 16 * 10 / ms / 1e6);
  cudaEventRecord(e0);
  for (int w = 0; w < 10; ++w) cudaMemcpyAsync(out, out + B * nq_s * 8, B * nq_s * 8, cudaMemcpyDeviceToDevice);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("memcpy d2d (read+write): %.1f GB/s\n", (double)B * nq_s * 16 * 10 / ms / 1e6);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
