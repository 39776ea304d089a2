// Per-SM L2 -> shared-memory ingest ceiling on B200 (the bound of the act GEMM's operand
// traffic and of the fused learner's tile loads): every CTA (one per SM) streams a window of
// an L2-resident buffer into shared memory, (a) with cp.async.bulk (TMA 1-D bulk copies,
// mbarrier completion), (b) with 16-byte cp.async from 256 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_ingest l2_ingest.cu && ./l2_ingest
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChunk = 32 * 1024;  // bytes per bulk copy / per cp.async round
constexpr int kStages = 4;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256) bulk_kernel(const char* __restrict__ src, size_t window, int rounds,
                                                   unsigned long long* cyc) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[kStages];
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* base = src + (size_t)blockIdx.x * window;
  const size_t nchunks = window / kChunk;
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    uint32_t phase[kStages] = {0, 0, 0, 0};
    for (long long it = 0; it < (long long)rounds * nchunks; ++it) {
      const int s = it % kStages;
      if (it >= kStages) {  // wait for the stage's previous copy
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(phase[s]));
        phase[s] ^= 1;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(kChunk));
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sm + s * kChunk)),
          "l"(base + (it % nchunks) * kChunk), "r"(kChunk), "r"(smem_u32(&bar[s]))
          : "memory");
    }
    for (int s = 0; s < kStages; ++s) {
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(smem_u32(&bar[s])), "r"(phase[s]));
    }
    cyc[blockIdx.x] = clock64() - t0;
  }
}

__global__ void __launch_bounds__(256) cpasync_kernel(const char* __restrict__ src, size_t window, int rounds,
                                                      unsigned long long* cyc) {
  extern __shared__ __align__(128) char sm[];
  const char* base = src + (size_t)blockIdx.x * window;
  const size_t nchunks = window / kChunk;
  long long t0 = clock64();
  for (long long it = 0; it < (long long)rounds * nchunks; ++it) {
    const char* g = base + (it % nchunks) * kChunk;
    char* d = sm + (it % kStages) * kChunk;
    for (int o = threadIdx.x * 16; o < kChunk; o += 256 * 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(d + o)), "l"(g + o) : "memory");
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 3;" ::: "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t window = 256 * 1024;  // per CTA: 148 x 256 KB = 37 MB, L2-resident
  char* buf;
  unsigned long long* cyc;
  cudaMalloc(&buf, window * sms);
  cudaMemset(buf, 1, window * sms);
  cudaMalloc(&cyc, 8 * sms);
  const int smem = kStages * kChunk;
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(cpasync_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rounds = 64;
  for (int mode = 0; mode < 2; ++mode) {
    for (int grid : {1, sms}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        if (mode == 0)
          bulk_kernel<<<grid, 256, smem>>>(buf, window, rounds, cyc);
        else
          cpasync_kernel<<<grid, 256, smem>>>(buf, window, rounds, cyc);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long h[256];
        cudaMemcpy(h, cyc, 8 * grid, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const double bytes = (double)window * rounds;
        if (rep == 1)
          printf("%-22s grid %3d: %.1f B/clk per SM (slowest CTA), %.0f GB/s per SM, aggregate %.0f GB/s (%s)\n",
                 mode == 0 ? "cp.async.bulk 32 KB" : "cp.async 16 B x 256 thr", grid, bytes / mx,
                 bytes / (ms * 1e-3) / 1e9, bytes * grid / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
