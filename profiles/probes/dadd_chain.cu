// Latency of a dependent fp64 add chain on B200 (the PER sampler's cumsum is one such chain).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dadd_chain dadd_chain.cu && ./dadd_chain
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(const double* x, double* out, long long* cyc, int n, int mode) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = x[i];
  __syncthreads();
  if (threadIdx.x) return;
  long long t0 = clock64();
  double acc = s[0];
  if (mode == 0) {  // register-only chain: acc + constant
    const double c = x[1];
    for (int i = 1; i < n; ++i) acc = acc + c;
  } else if (mode == 1) {  // cumsum from shared memory, stores back
    for (int i = 1; i < n; i += 16) {
      double v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = s[i + k];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        acc = acc + v[k];
        s[i + k] = acc;
      }
    }
  } else {  // cumsum from global memory (L2), 16 at a time
    for (int i = 1; i < n; i += 16) {
      double v[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = x[i + k];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        acc = acc + v[k];
        out[i + k] = acc;
      }
    }
  }
  long long t1 = clock64();
  out[0] = acc;
  *cyc = t1 - t0;
}

int main() {
  const int n = 2001;
  double *x, *out;
  long long* cyc;
  cudaMalloc(&x, 8 * 4096);
  cudaMalloc(&out, 8 * 4096);
  cudaMalloc(&cyc, 8);
  double h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = 1.0 / (i + 3);
  cudaMemcpy(x, h, sizeof h, cudaMemcpyHostToDevice);
  const char* names[] = {"register chain", "cumsum smem", "cumsum global"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) chain<<<1, 256>>>(x, out, cyc, n, mode);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    chain<<<1, 256>>>(x, out, cyc, n, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-16s n=%d: %lld cycles (%.2f per add), kernel %.2f us\n", names[mode], n - 1, c, (double)c / (n - 1),
           ms * 1e3);
  }
  return 0;
}
