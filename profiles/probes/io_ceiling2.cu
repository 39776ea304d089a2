// Write-path ceilings: SM 16-byte stores vs TMA bulk stores (smem -> global),
// for K1's 5648-byte slot rows (+ its 1072-byte seed reads).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_cs(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void stg(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// flat write-only, 16 B per thread per iteration
template <bool CS>
__global__ void flat_write(int8_t* out, int64_t n16) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n16; i += nt) {
    if (CS) stg_cs(out + 16 * i, make_uint4(i, 1, 2, 3));
    else stg(out + 16 * i, make_uint4(i, 1, 2, 3));
  }
}

// warp per plan row; the warp stages a row in smem and one lane issues a bulk store.
// NBUF row buffers per warp so the bulk stores overlap the next rows.
template <int NBUF, bool READ>
__global__ void __launch_bounds__(256) bulk_rows(const int8_t* seeds, int64_t ss, int nq_d, int8_t* out, int64_t os,
                                                 int row_bytes, int64_t batch) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint8_t* mybuf = smem + (size_t)warp * NBUF * os;
  const int64_t nw = (int64_t)gridDim.x * 8;
  int k = 0;
  for (int64_t b = blockIdx.x * 8 + warp; b < batch; b += nw, k = (k + 1) % NBUF) {
    uint32_t x = 0;
    if (READ) {
      for (int q = lane; q < nq_d; q += 32) {
        uint4 v = ldg_stream(seeds + b * ss + 16 * q);
        x ^= v.x ^ v.w;
      }
      x = __reduce_or_sync(0xffffffffu, x);
    }
    // wait until buffer k's previous bulk store has read smem
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
    __syncwarp();
    uint4* row = reinterpret_cast<uint4*>(mybuf + (size_t)k * os);
    for (int q = lane; q < row_bytes / 16; q += 32) row[q] = make_uint4(x, q, 2, 3);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const uint32_t sa = (uint32_t)__cvta_generic_to_shared(row);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + b * os), "r"(sa),
                   "r"(row_bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// SM-store reference with the same structure (warp per row, 16 B stores)
template <bool READ>
__global__ void __launch_bounds__(256) stg_rows(const int8_t* seeds, int64_t ss, int nq_d, int8_t* out, int64_t os,
                                                int row_bytes, int64_t batch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t b = blockIdx.x * 8 + warp; b < batch; b += nw) {
    uint32_t x = 0;
    if (READ) {
      for (int q = lane; q < nq_d; q += 32) {
        uint4 v = ldg_stream(seeds + b * ss + 16 * q);
        x ^= v.x ^ v.w;
      }
      x = __reduce_or_sync(0xffffffffu, x);
    }
    for (int q = lane; q < row_bytes / 16; q += 32) stg_cs(out + b * os + 16 * q, make_uint4(x, q, 2, 3));
  }
}

static float timeit(void (*launch)(void*), void* ctx) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) launch(ctx);
  cudaEventRecord(e0);
  for (int w = 0; w < 20; ++w) launch(ctx);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 20;
}

struct Ctx {
  int8_t *seeds, *out;
  int64_t B;
  int sms, nq_d, nq_s, per_sm;
};

int main() {
  const int D = 1059, S = 5633;
  Ctx c;
  c.nq_d = (D + 15) / 16;
  c.nq_s = (S + 15) / 16;
  c.B = 1 << 22;
  cudaMalloc(&c.seeds, c.B * c.nq_d * 16);
  cudaMalloc(&c.out, c.B * c.nq_s * 16);
  cudaMemset(c.seeds, 1, c.B * c.nq_d * 16);
  cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, 0);
  const double wbytes = (double)c.B * c.nq_s * 16, rbytes = (double)c.B * c.nq_d * 16;
  for (int per_sm : {4, 8}) {
    c.per_sm = per_sm;
    float ms = timeit([](void* p) {
      Ctx* c = (Ctx*)p;
      flat_write<true><<<c->sms * c->per_sm, 256>>>(c->out, c->B * c->nq_s);
    }, &c);
    printf("flat write .cs   ctas/sm=%d: %.1f GB/s\n", per_sm, wbytes / ms / 1e6);
    ms = timeit([](void* p) {
      Ctx* c = (Ctx*)p;
      flat_write<false><<<c->sms * c->per_sm, 256>>>(c->out, c->B * c->nq_s);
    }, &c);
    printf("flat write plain ctas/sm=%d: %.1f GB/s\n", per_sm, wbytes / ms / 1e6);
  }
  for (int per_sm : {2, 4}) {
    c.per_sm = per_sm;
    float ms = timeit([](void* p) {
      Ctx* c = (Ctx*)p;
      stg_rows<false><<<c->sms * c->per_sm, 256>>>(c->seeds, c->nq_d * 16, c->nq_d, c->out, c->nq_s * 16, c->nq_s * 16, c->B);
    }, &c);
    printf("stg rows write-only   ctas/sm=%d: %.1f GB/s\n", per_sm, wbytes / ms / 1e6);
    ms = timeit([](void* p) {
      Ctx* c = (Ctx*)p;
      stg_rows<true><<<c->sms * c->per_sm, 256>>>(c->seeds, c->nq_d * 16, c->nq_d, c->out, c->nq_s * 16, c->nq_s * 16, c->B);
    }, &c);
    printf("stg rows read+write   ctas/sm=%d: %.1f GB/s (%.1f M rows/s)\n", per_sm, (wbytes + rbytes) / ms / 1e6,
           c.B / ms / 1e3);
  }
  const int smem2 = 8 * 2 * c.nq_s * 16, smem3 = 8 * 3 * c.nq_s * 16;
  cudaFuncSetAttribute(bulk_rows<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
  cudaFuncSetAttribute(bulk_rows<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
  cudaFuncSetAttribute(bulk_rows<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
  for (int per_sm : {1, 2}) {
    c.per_sm = per_sm;
    float ms = timeit([](void* p) {
      Ctx* c = (Ctx*)p;
      bulk_rows<2, false><<<c->sms * c->per_sm, 256, 8 * 2 * c->nq_s * 16>>>(c->seeds, c->nq_d * 16, c->nq_d, c->out,
                                                                          c->nq_s * 16, c->nq_s * 16, c->B);
    }, &c);
    printf("bulk rows write-only NBUF=2 ctas/sm=%d: %.1f GB/s\n", per_sm, wbytes / ms / 1e6);
    ms = timeit([](void* p) {
      Ctx* c = (Ctx*)p;
      bulk_rows<2, true><<<c->sms * c->per_sm, 256, 8 * 2 * c->nq_s * 16>>>(c->seeds, c->nq_d * 16, c->nq_d, c->out,
                                                                         c->nq_s * 16, c->nq_s * 16, c->B);
    }, &c);
    printf("bulk rows read+write NBUF=2 ctas/sm=%d: %.1f GB/s (%.1f M rows/s)\n", per_sm,
           (wbytes + rbytes) / ms / 1e6, c.B / ms / 1e3);
    ms = timeit([](void* p) {
      Ctx* c = (Ctx*)p;
      bulk_rows<3, true><<<c->sms * c->per_sm, 256, 8 * 3 * c->nq_s * 16>>>(c->seeds, c->nq_d * 16, c->nq_d, c->out,
                                                                         c->nq_s * 16, c->nq_s * 16, c->B);
    }, &c);
    printf("bulk rows read+write NBUF=3 ctas/sm=%d: %.1f GB/s (%.1f M rows/s)\n", per_sm,
           (wbytes + rbytes) / ms / 1e6, c.B / ms / 1e3);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
