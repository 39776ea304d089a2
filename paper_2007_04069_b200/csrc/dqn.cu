// DQN learner kernels (reference agent.py:58-337), device-resident.
//
// The Q-network GEMMs run on the tensor cores (gemm_tc.cu); these kernels are
// the non-GEMM parts, each fused to one pass:
//   dueling combine          Q = V + A - mean(A)                (agent.py:104-109)
//   masked argmax / act      ties to the lowest index           (agent.py:147-170)
//   TD + Huber + head grads  double-DQN target, IS weights,     (agent.py:258-299)
//                            dQ folded straight into dV / dA    (agent.py:114-118)
//   ReLU backward, column sums (bias grads)                     (agent.py:119-136)
//   Adam with bias correction over one flat parameter buffer    (agent.py:229-250)
//   PER: priority**alpha, numpy pairwise sum, sequential cumsum,
//        searchsorted(side='right'), IS weights; last-write-wins
//        priority scatter                                        (agent.py:183-226)
// PER arithmetic is fp64 and follows numpy's evaluation order so the sampled
// indices match the reference for the same uniforms.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "engine.h"
#include "per_sample.cuh"

namespace apb {

bool pdl_enabled() { return std::getenv("AP_NO_PDL") == nullptr; }

namespace {

constexpr unsigned kFull = 0xffffffffu;

// Q = V + A - mean(A), one warp per row.  Loads are issued 4 deep ahead of the
// adds (each lane's add order is unchanged); z and q never alias.
__global__ void dueling_kernel(const float* __restrict__ z, int64_t ldz, float* __restrict__ q, int64_t ldq, int B,
                               int A) {
  pdl_entry();
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  const float* __restrict__ row = z + (int64_t)b * ldz + 1;
  float* __restrict__ out = q + (int64_t)b * ldq;
  float s = 0.0f;
  int j = lane;
  for (; j + 96 < A; j += 128) {
    const float x0 = row[j], x1 = row[j + 32], x2 = row[j + 64], x3 = row[j + 96];
    s += x0;
    s += x1;
    s += x2;
    s += x3;
  }
  for (; j < A; j += 32) s += row[j];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  const float mean = s / (float)A;
  const float v = z[(int64_t)b * ldz];
#pragma unroll 4
  for (int k = lane; k < A; k += 32) out[k] = v + row[k] - mean;
}

// Wide action spaces (A > 256): one 256-thread CTA per row (a warp per row
// leaves too few loads in flight when A is in the thousands and B is small).
__global__ void __launch_bounds__(256) dueling_wide_kernel(const float* __restrict__ z, int64_t ldz,
                                                           float* __restrict__ q, int64_t ldq, int B, int A) {
  pdl_entry();
  __shared__ float s_part[8];
  const int b = blockIdx.x;
  const float* __restrict__ row = z + (int64_t)b * ldz + 1;
  float* __restrict__ out = q + (int64_t)b * ldq;
  float s = 0.0f;
  int j = threadIdx.x;
  for (; j + 768 < A; j += 1024) {
    const float x0 = row[j], x1 = row[j + 256], x2 = row[j + 512], x3 = row[j + 768];
    s += x0;
    s += x1;
    s += x2;
    s += x3;
  }
  for (; j < A; j += 256) s += row[j];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = s;
  __syncthreads();
  float tot = 0.0f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += s_part[w];
  const float mean = tot / (float)A;
  const float v = z[(int64_t)b * ldz];
#pragma unroll 4
  for (int k = threadIdx.x; k < A; k += 256) out[k] = v + row[k] - mean;
}

// masked argmax (ties -> lowest index); eps-greedy with a counter-based hash
// when eps > 0 (throughput mode; parity mode draws on the host)
__device__ inline uint32_t hash32(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return (uint32_t)x;
}

// Linear epsilon decay (agent.py:50-55) from the device train-step counter.
__device__ inline float epsilon_dev(int64_t it, float e0, float e1, int64_t decay) {
  if (decay <= 0) return e1;
  const double frac = fmin(1.0, fmax(0.0, (double)it / (double)decay));
  return (float)((double)e0 + ((double)e1 - (double)e0) * frac);
}

// ctl != nullptr (graph-capturable driver): epsilon from ctl[AP_CTL_TRAIN], hash
// counter ctl[AP_CTL_STEP] + 1, instead of the by-value arguments
__global__ void act_kernel(const float* q, int64_t ldq, const uint8_t* mask, int64_t ldm, int E, int A, float eps,
                           uint64_t seed, int32_t* out, const int64_t* ctl, float eps0, float eps1, int64_t decay) {
  pdl_entry();
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= E) return;
  if (ctl) {
    eps = epsilon_dev(ctl[AP_CTL_TRAIN], eps0, eps1, decay);
    seed = (uint64_t)ctl[AP_CTL_STEP] + 1;
  }
  const uint8_t* __restrict__ m = mask + (int64_t)e * ldm;
  const float* __restrict__ qr = q + (int64_t)e * ldq;
  int count = 0;
  float best = -INFINITY;
  int best_j = 0x7fffffff;
  auto visit = [&](int j, uint8_t ok, float v) {
    if (!ok) return;
    ++count;
    if (v > best || (v == best && j < best_j)) {
      best = v;
      best_j = j;
    }
  };
  int j = lane;
  for (; j + 96 < A; j += 128) {  // 4 rows of loads in flight, visited in ascending j
    uint8_t ok[4];
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      ok[u] = m[j + 32 * u];
      v[u] = qr[j + 32 * u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) visit(j + 32 * u, ok[u], v[u]);
  }
  for (; j < A; j += 32) visit(j, m[j], qr[j]);
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(kFull, best, o);
    const int oj = __shfl_xor_sync(kFull, best_j, o);
    if (ov > best || (ov == best && oj < best_j)) {
      best = ov;
      best_j = oj;
    }
    count += __shfl_xor_sync(kFull, count, o);
  }
  int action = best_j == 0x7fffffff ? -1 : best_j;
  if (eps > 0.0f && count > 0) {
    const uint32_t r0 = hash32(seed * 0x9E3779B97F4A7C15ULL + (uint64_t)e * 2 + 0);
    if ((float)(r0 >> 8) * (1.0f / 16777216.0f) < eps) {
      const int pick = (int)(hash32(seed * 0x9E3779B97F4A7C15ULL + (uint64_t)e * 2 + 1) % (uint32_t)count);
      // the pick-th allowed action
      int seen = 0;
      action = -1;
      for (int base = 0; base < A && action < 0; base += 32) {
        const int j = base + lane;
        const bool ok = j < A && m[j];
        const unsigned bal = __ballot_sync(kFull, ok);
        const int n = __popc(bal);
        if (pick < seen + n) {
          unsigned bits = bal;
          for (int k = 0; k < pick - seen; ++k) bits &= bits - 1;
          action = base + __ffs(bits) - 1;
        }
        seen += n;
      }
    }
  }
  if (lane == 0) out[e] = action;
}

// Double-DQN TD error, Huber-weighted loss and the gradient w.r.t. the fused
// head outputs z = [V, A_0..A_{n-1}] (agent.py:258-299, 114-118).
// idx != nullptr: the transition fields are read from replay-ring rows idx[b]
// (fused gather); dz_t != nullptr: also writes dz^T [1 + A, B] (the K-major
// operand of the head weight-gradient GEMM)
__global__ void td_kernel(const float* q, const float* online_next, const float* target_next, int64_t ldq,
                          const int32_t* actions, const float* rewards, const uint8_t* done, const uint8_t* next_mask,
                          int64_t ldm, const float* weights, int B, int A, float gamma, float delta, float* dz,
                          int64_t ldz, float* td_out, float* loss_out, const int32_t* idx, float* dz_t,
                          int64_t ldzt) {
  pdl_entry();
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  const int64_t row = idx ? (int64_t)idx[b] : (int64_t)b;
  const uint8_t* m = next_mask + row * ldm;
  // best next action by the online net over the (safe) next mask
  bool any = false;
  float best = -INFINITY;
  int best_j = 0x7fffffff;
  for (int j = lane; j < A; j += 32) {
    if (!m[j]) continue;
    any = true;
    const float v = online_next[(int64_t)b * ldq + j];
    if (v > best || (v == best && j < best_j)) {
      best = v;
      best_j = j;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(kFull, best, o);
    const int oj = __shfl_xor_sync(kFull, best_j, o);
    if (ov > best || (ov == best && oj < best_j)) {
      best = ov;
      best_j = oj;
    }
  }
  any = __any_sync(kFull, any);
  const int a_next = any ? best_j : 0;  // empty mask: action 0 is "safe", bootstrap zeroed below
  const float d = (done[row] || !any) ? 1.0f : 0.0f;
  const float target = rewards[row] + gamma * (1.0f - d) * target_next[(int64_t)b * ldq + a_next];
  const int a = actions[row];
  const float td = q[(int64_t)b * ldq + a] - target;
  const float w = weights[b];
  const float ad = fabsf(td);
  const float hub = ad <= delta ? 0.5f * td * td : delta * (ad - 0.5f * delta);
  const float g = w * fminf(fmaxf(td, -delta), delta) / (float)B;
  for (int j = lane; j <= A; j += 32) {
    float v;
    if (j == 0)
      v = g;  // dV = sum_j dQ_j
    else
      v = ((j - 1) == a ? g : 0.0f) - g / (float)A;  // dA_j = dQ_j - sum(dQ)/A
    dz[(int64_t)b * ldz + j] = v;
    if (dz_t) dz_t[(int64_t)j * ldzt + b] = v;
  }
  if (lane == 0) {
    td_out[b] = td;
    loss_out[b] = w * hub;  // loss = mean over rows, reduced deterministically by the caller
  }
}

// Dueling head forward for narrow heads (1 + A <= kHeadMax outputs): one warp
// per row computes z = h @ wh + bh (wh given transposed, [1 + A, H]) with the
// lanes splitting H, then Q = V + A - mean(A) (agent.py:99-109).
constexpr int kHeadMax = 8;

template <int A1>
__global__ void head_forward_kernel(const float* h, int64_t ldh, const float* wht, int64_t ldw, const float* bh,
                                    int B, int H, float* q, int64_t ldq) {
  pdl_entry();
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= B) return;
  float z[A1];
#pragma unroll
  for (int j = 0; j < A1; ++j) z[j] = 0.0f;
  const float* hr = h + (int64_t)b * ldh;
  for (int k = lane; k < H; k += 32) {
    const float x = hr[k];
#pragma unroll
    for (int j = 0; j < A1; ++j) z[j] = fmaf(x, wht[(int64_t)j * ldw + k], z[j]);
  }
#pragma unroll
  for (int j = 0; j < A1; ++j)
    for (int o = 16; o; o >>= 1) z[j] += __shfl_xor_sync(kFull, z[j], o);
  if (lane == 0) {
    float mean = 0.0f;
#pragma unroll
    for (int j = 0; j < A1; ++j) z[j] += bh[j];
#pragma unroll
    for (int j = 1; j < A1; ++j) mean += z[j];
    mean /= (float)(A1 - 1);
#pragma unroll
    for (int j = 1; j < A1; ++j) q[(int64_t)b * ldq + (j - 1)] = z[0] + z[j] - mean;
  }
}

// td_kernel for wide action spaces (PP): one CTA per row, the masked argmax
// over the next-state Q and the dz row writes spread over the CTA's threads.
// Same arithmetic and tie rules as td_kernel.
__global__ void td_wide_kernel(const float* q, const float* online_next, const float* target_next, int64_t ldq,
                               const int32_t* actions, const float* rewards, const uint8_t* done,
                               const uint8_t* next_mask, int64_t ldm, const float* weights, int B, int A, float gamma,
                               float delta, float* dz, int64_t ldz, float* td_out, float* loss_out, const int32_t* idx,
                               float* dz_t, int64_t ldzt) {
  pdl_entry();
  __shared__ float s_best[32];
  __shared__ int s_bj[32], s_any[32];
  __shared__ float s_g;
  __shared__ int s_a;
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t row = idx ? (int64_t)idx[b] : (int64_t)b;
  const uint8_t* __restrict__ m = next_mask + row * ldm;
  const float* __restrict__ on = online_next + (int64_t)b * ldq;
  float best = -INFINITY;
  int best_j = 0x7fffffff, any = 0;
  auto visit = [&](int j, uint8_t ok, float v) {
    if (!ok) return;
    any = 1;
    if (v > best || (v == best && j < best_j)) {
      best = v;
      best_j = j;
    }
  };
  const int st = blockDim.x;
  int j = threadIdx.x;
  for (; j + 3 * st < A; j += 4 * st) {  // 4 loads in flight per thread
    uint8_t ok[4];
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      ok[u] = m[j + u * st];
      v[u] = on[j + u * st];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) visit(j + u * st, ok[u], v[u]);
  }
  for (; j < A; j += st) visit(j, m[j], on[j]);
  for (int o = 16; o; o >>= 1) {
    const float ov = __shfl_xor_sync(kFull, best, o);
    const int oj = __shfl_xor_sync(kFull, best_j, o);
    if (ov > best || (ov == best && oj < best_j)) {
      best = ov;
      best_j = oj;
    }
    any |= __shfl_xor_sync(kFull, any, o);
  }
  if (lane == 0) {
    s_best[warp] = best;
    s_bj[warp] = best_j;
    s_any[warp] = any;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w) {
      if (s_best[w] > best || (s_best[w] == best && s_bj[w] < best_j)) {
        best = s_best[w];
        best_j = s_bj[w];
      }
      any |= s_any[w];
    }
    const int a_next = any ? best_j : 0;  // empty mask: action 0 is "safe", bootstrap zeroed below
    const float d = (done[row] || !any) ? 1.0f : 0.0f;
    const float target = rewards[row] + gamma * (1.0f - d) * target_next[(int64_t)b * ldq + a_next];
    const int a = actions[row];
    const float td = q[(int64_t)b * ldq + a] - target;
    const float w = weights[b];
    const float ad = fabsf(td);
    const float hub = ad <= delta ? 0.5f * td * td : delta * (ad - 0.5f * delta);
    s_g = w * fminf(fmaxf(td, -delta), delta) / (float)B;
    s_a = a;
    td_out[b] = td;
    loss_out[b] = w * hub;
  }
  __syncthreads();
  const float g = s_g;
  const int a = s_a;
  for (int j = threadIdx.x; j <= A; j += blockDim.x) {
    const float v = j == 0 ? g : (((j - 1) == a ? g : 0.0f) - g / (float)A);
    dz[(int64_t)b * ldz + j] = v;
    if (dz_t) dz_t[(int64_t)j * ldzt + b] = v;
  }
}

// Up to 8 matrix transposes in one launch (the transposed weight copies the
// K-major GEMMs read, refreshed after every Adam step): blockIdx.z = segment,
// 32x32 tiles staged through shared memory so both sides are coalesced.
struct TransposeBatch {
  const float* src[8];
  float* dst[8];
  int64_t lds[8], ldd[8];
  int32_t rows[8], cols[8];
};

__global__ void transpose_batch_kernel(TransposeBatch tb) {
  pdl_entry();
  __shared__ float tile[32][33];
  const int z = blockIdx.z;
  const int rows = tb.rows[z], cols = tb.cols[z];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  if (r0 >= rows || c0 >= cols) return;
  const float* src = tb.src[z];
  float* dst = tb.dst[z];
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = src[(int64_t)r * tb.lds[z] + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) dst[(int64_t)c * tb.ldd[z] + r] = tile[threadIdx.x][k];
  }
}

// ReLU backward in place on dh [B, H] plus the transposed copy dh_t [H, B]
// (the K-major operand of the next weight-gradient GEMM)
__global__ void relu_bwd_t_kernel(float* dh, int64_t lddh, const float* h, int64_t ldh, int B, int H, float* dh_t,
                                  int64_t ldt) {
  pdl_entry();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * H) return;
  const int b = (int)(i / H), j = (int)(i % H);
  float v = dh[(int64_t)b * lddh + j];
  if (!(h[(int64_t)b * ldh + j] > 0.0f)) {
    v = 0.0f;
    dh[(int64_t)b * lddh + j] = 0.0f;
  }
  dh_t[(int64_t)j * ldt + b] = v;
}

__global__ void relu_bwd_kernel(float* dh, const float* h, int64_t n) {
  pdl_entry();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!(h[i] > 0.0f)) dh[i] = 0.0f;
}

// Gradient into the last hidden layer from the (1 + A)-wide dueling head
// (agent.py:120-129): dh = relu'(h) * (dz @ wh^T), a K = 1 + A contraction too
// narrow for the tensor cores; optionally also dh^T (the next weight-gradient
// GEMM's K-major operand).  One thread per (row, unit).
__global__ void head_backward_kernel(const float* dz, int64_t ldz, const float* wh, int64_t ldw, const float* h,
                                     int64_t ldh, int B, int H, int A1, float* dh, int64_t lddh, float* dh_t,
                                     int64_t ldt) {
  pdl_entry();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * H) return;
  const int b = (int)(i / H), j = (int)(i % H);
  float acc = 0.0f;
  for (int k = 0; k < A1; ++k) acc = fmaf(dz[(int64_t)b * ldz + k], wh[(int64_t)j * ldw + k], acc);
  if (!(h[(int64_t)b * ldh + j] > 0.0f)) acc = 0.0f;
  dh[(int64_t)b * lddh + j] = acc;
  if (dh_t) dh_t[(int64_t)j * ldt + b] = acc;
}

// Wide-head variant: a warp per (row, unit) with the lanes striding the 1 + A
// head outputs (coalesced reads of the dz row and of the unit's wh row), then a
// shuffle reduction.
// Dueling-structured head backward (throughput learner): the TD kernels write
// dz[b] = g_b * (e_0 + e_{1+a_b}) - (g_b / A) * [0, 1, .., 1], so
//   dh[b, j] = g_b * wh[j, 0] + g_b * wh[j, 1 + a_b] - (g_b / A) * rowsum_j,
// rowsum_j = sum_k wh[j, 1 + k] (head_rowsum_kernel, once per backward).
// a_b is the one advantage entry that differs from 0 - g_b/A (the TD kernels'
// own expression, so the comparison is exact); g_b == 0 gives dh = 0.
__global__ void __launch_bounds__(256) head_rowsum_kernel(const float* __restrict__ wh, int64_t ldw, int A1,
                                                          float* __restrict__ rowsum) {
  pdl_entry();
  __shared__ float s_part[8];
  const float* __restrict__ w = wh + (int64_t)blockIdx.x * ldw;
  float s = 0.0f;
  for (int k = 1 + threadIdx.x; k < A1; k += 256) s += w[k];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.0f;
    for (int k = 0; k < 8; ++k) t += s_part[k];
    rowsum[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(256) head_backward_dueling_kernel(const float* __restrict__ dz, int64_t ldz,
                                                                    const float* __restrict__ wh, int64_t ldw,
                                                                    const float* __restrict__ h, int64_t ldh,
                                                                    const float* __restrict__ rowsum, int H, int A1,
                                                                    float* __restrict__ dh, int64_t lddh,
                                                                    float* __restrict__ dh_t, int64_t ldt) {
  pdl_entry();
  __shared__ int s_a, s_cnt, s_nz;
  const int b = blockIdx.x;
  const int A = A1 - 1;
  const float* __restrict__ z = dz + (int64_t)b * ldz;
  const float g = z[0];
  const float other = 0.0f - g / (float)A;
  if (threadIdx.x == 0) {
    s_a = 0;
    s_cnt = 0;
    s_nz = 0;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < A; k += blockDim.x) {
    const float x = z[1 + k];
    if (x != other) {
      s_a = k;
      atomicAdd(&s_cnt, 1);
    }
    if (x != 0.0f) s_nz = 1;
  }
  __syncthreads();
  const int a = s_a;
  // rows not of the TD shape (never produced by the TD kernels) take the full product
  const bool closed = g != 0.0f ? s_cnt == 1 : s_nz == 0;
  const float ga = g / (float)A;
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    const float* __restrict__ w = wh + (int64_t)j * ldw;
    float acc;
    if (closed) {
      acc = g == 0.0f ? 0.0f : g * w[0] + g * w[1 + a] - ga * rowsum[j];
    } else {
      acc = 0.0f;
      for (int k = 0; k < A1; ++k) acc = fmaf(z[k], w[k], acc);
    }
    if (!(h[(int64_t)b * ldh + j] > 0.0f)) acc = 0.0f;
    dh[(int64_t)b * lddh + j] = acc;
    if (dh_t) dh_t[(int64_t)j * ldt + b] = acc;
  }
}

__global__ void head_backward_wide_kernel(const float* dz, int64_t ldz, const float* wh, int64_t ldw, const float* h,
                                          int64_t ldh, int B, int H, int A1, float* dh, int64_t lddh, float* dh_t,
                                          int64_t ldt) {
  pdl_entry();
  const int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= (int64_t)B * H) return;
  const int b = (int)(w / H), j = (int)(w % H);
  const float* zr = dz + (int64_t)b * ldz;
  const float* wr = wh + (int64_t)j * ldw;
  float acc = 0.0f;
  for (int k = lane; k < A1; k += 32) acc = fmaf(zr[k], wr[k], acc);
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
  if (lane == 0) {
    if (!(h[(int64_t)b * ldh + j] > 0.0f)) acc = 0.0f;
    dh[(int64_t)b * lddh + j] = acc;
    if (dh_t) dh_t[(int64_t)j * ldt + b] = acc;
  }
}

__global__ void colsum_kernel(const float* x, int64_t ld, int rows, int cols, float* out) {
  pdl_entry();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.0f;
  for (int r = 0; r < rows; ++r) s += x[(int64_t)r * ld + c];
  out[c] = s;
}

// ctl != nullptr: bias corrections from step t = ctl[AP_CTL_TRAIN] + 1
__global__ void adam_kernel(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                            float eps, float c1, float c2, const int64_t* ctl, const float* ctab,
                            int64_t t_offset) {
  pdl_entry();
  if (ctab) {  // parity loop: the host's fp32(1 - beta**t), t = ctl[AP_CTL_TRAIN] + t_offset + 1
    const int64_t k = ctl[AP_CTL_TRAIN] + t_offset - ctl[AP_PL_TAB_BASE];
    c1 = ctab[2 * k];
    c2 = ctab[2 * k + 1];
  } else if (ctl) {  // bias corrections once per block, not per thread (two fp64 pow)
    __shared__ float s_c[2];
    if (threadIdx.x == 0) {
      const double t = (double)(ctl[AP_CTL_TRAIN] + 1);
      s_c[0] = (float)(1.0 - pow((double)b1, t));
      s_c[1] = (float)(1.0 - pow((double)b2, t));
    }
    __syncthreads();
    c1 = s_c[0];
    c2 = s_c[1];
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.0f - b1) * gi;
    const float vi = b2 * v[i] + (1.0f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
  }
}

// Adam (control-block step count) that also refreshes the transposed weight
// copies the K-major GEMMs read: element i of segment s (flat offset off[s],
// [rows, cols] row-major) is written to dst[s][c * ldd[s] + r] as well, so no
// separate transpose launch follows the update.
struct AdamSegments {
  int64_t off[8];
  int32_t rows[8], cols[8];
  float* dst[8];
  int64_t ldd[8];
  int n;
  int t_add;  // Adam step t = ctl[AP_CTL_TRAIN] + t_add (0 when the counter was already advanced)
};

// one Adam element update (shared by the flat and tiled kernels: same code, same rounding)
__device__ __forceinline__ float adam_elem(float* p, const float* g, float* m, float* v, int64_t i, float lr, float b1,
                                           float b2, float eps, float c1, float c2) {
  float mi = m[i], vi = v[i], pi = p[i];
  adam_math(g[i], mi, vi, pi, lr, b1, b2, eps, c1, c2);
  m[i] = mi;
  v[i] = vi;
  p[i] = pi;
  return pi;
}

// Tiled adam_t: one 256-thread block per 32x32 tile of a weight segment
// (coalesced reads / writes of p, g, m, v; the transposed copy goes out
// through a shared-memory tile, coalesced as well), then flat blocks over the
// elements outside every segment (biases).  tile_base / gap ranges are built
// on the host; segments are disjoint.
struct AdamTiles {
  AdamSegments segs;
  int64_t tile_base[9];
  int32_t tcols[8];
  int64_t gap_lo[9], gap_base[10];
  int ngap;
};

__global__ void __launch_bounds__(256) adam_tile_kernel(float* p, const float* g, float* m, float* v, float lr,
                                                        float b1, float b2, float eps, const int64_t* ctl,
                                                        AdamTiles at) {
  pdl_entry();
  __shared__ float s_c[2];
  __shared__ float tile[32][33];
  auto corrections = [&]() {  // bias corrections (thread 0), published by the caller's barrier
    if (threadIdx.x == 0) {
      const double t = (double)(ctl[AP_CTL_TRAIN] + at.segs.t_add);
      s_c[0] = (float)(1.0 / (1.0 - pow((double)b1, t)));
      s_c[1] = (float)(1.0 / (1.0 - pow((double)b2, t)));
    }
  };
  const int64_t ntiles = at.tile_base[at.segs.n];
  const int64_t blk = blockIdx.x;
  if (blk < ntiles) {
    int s = 0;
    while (blk >= at.tile_base[s + 1]) ++s;
    const int64_t t = blk - at.tile_base[s];
    const int tr = (int)(t / at.tcols[s]), tc = (int)(t % at.tcols[s]);
    const int rows = at.segs.rows[s], cols = at.segs.cols[s];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t off = at.segs.off[s];
    // the tile's loads go out before the (pow-latency) bias corrections are awaited
    float gv[4], mv[4], vv[4], pv[4];
    int64_t ix[4];
    bool ok[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int r = tr * 32 + ty + 8 * k, c = tc * 32 + tx;
      ok[k] = r < rows && c < cols;
      ix[k] = off + (int64_t)r * cols + c;
      if (ok[k]) {
        gv[k] = g[ix[k]];
        mv[k] = m[ix[k]];
        vv[k] = v[ix[k]];
        pv[k] = p[ix[k]];
      }
    }
    corrections();
    __syncthreads();
    const float c1 = s_c[0], c2 = s_c[1];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (ok[k]) {
        adam_math(gv[k], mv[k], vv[k], pv[k], lr, b1, b2, eps, c1, c2);
        m[ix[k]] = mv[k];
        v[ix[k]] = vv[k];
        p[ix[k]] = pv[k];
        tile[ty + 8 * k][tx] = pv[k];
      }
    }
    __syncthreads();
    float* dst = at.segs.dst[s];
    const int64_t ldd = at.segs.ldd[s];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int c = tc * 32 + ty + 8 * k, r = tr * 32 + tx;  // dst[c][r] = w[r][c]
      if (r < rows && c < cols) dst[(int64_t)c * ldd + r] = tile[tx][ty + 8 * k];
    }
    return;
  }
  corrections();
  __syncthreads();
  const float c1 = s_c[0], c2 = s_c[1];
  const int64_t idx = (blk - ntiles) * blockDim.x + threadIdx.x;
  if (idx >= at.gap_base[at.ngap]) return;
  int q = 0;
  while (idx >= at.gap_base[q + 1]) ++q;
  adam_elem(p, g, m, v, at.gap_lo[q] + (idx - at.gap_base[q]), lr, b1, b2, eps, c1, c2);
}

__global__ void adam_t_kernel(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                              float eps, const int64_t* ctl, AdamSegments segs) {
  pdl_entry();
  __shared__ float s_c[2];
  if (threadIdx.x == 0) {
    const double t = (double)(ctl[AP_CTL_TRAIN] + segs.t_add);
    s_c[0] = (float)(1.0 / (1.0 - pow((double)b1, t)));  // reciprocals (adam_math)
    s_c[1] = (float)(1.0 / (1.0 - pow((double)b2, t)));
  }
  __syncthreads();
  const float c1 = s_c[0], c2 = s_c[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float pi = adam_elem(p, g, m, v, i, lr, b1, b2, eps, c1, c2);
    for (int s = 0; s < segs.n; ++s) {
      const int64_t rel = i - segs.off[s];
      if (rel >= 0 && rel < (int64_t)segs.rows[s] * segs.cols[s]) {
        const int64_t r = rel / segs.cols[s], c = rel % segs.cols[s];
        segs.dst[s][c * segs.ldd[s] + r] = pi;
        break;
      }
    }
  }
}

// one CTA: PER sample (agent.py:207-223) for B uniforms drawn by the caller (per_sample.cuh)
__global__ void __launch_bounds__(512) per_sample_kernel(const double* prio, int n, double alpha, double beta,
                                                         const double* uniforms, int B, double* scaled, double* cdf,
                                                         int32_t* idx_out, float* w_out, const int64_t* ctl) {
  pdl_entry();
  if (ctl) n = (int)ctl[AP_CTL_SIZE];  // device-held ring size (parity loop)
  if (ctl && n < B) return;            // no learn step yet (self-gated loop body)
  __shared__ PerShared S;
  per_sample_block(prio, n, alpha, beta, uniforms, B, scaled, cdf, idx_out, w_out, S);
}

// priorities[idx] = |td| + 1e-6, duplicates: the last occurrence wins (agent.py:226)
__global__ void per_update_kernel(double* prio, const int32_t* idx, const float* td, int B) {
  pdl_entry();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  for (int k = b + 1; k < B; ++k)
    if (idx[k] == idx[b]) return;
  prio[idx[b]] = fabs((double)td[b]) + 1e-6;
}

// dst[b, :cols] = src[idx[b], :cols]: blockIdx.y = b, 16-byte vectors when the
// rows and bases allow (no per-element index arithmetic)
// blockIdx.z selects one of up to two (src, dst) pairs gathered with the same indices
struct GatherPair {
  const float* src[2];
  int64_t lds[2];
  float* dst[2];
  int64_t ldd[2];
};

__global__ void gather_rows_kernel(GatherPair gp, const int32_t* __restrict__ idx, int B, int cols, int vec) {
  pdl_entry();
  const int b = blockIdx.y, z = blockIdx.z;
  const float* __restrict__ s = gp.src[z] + (int64_t)idx[b] * gp.lds[z];
  float* __restrict__ d = gp.dst[z] + (int64_t)b * gp.ldd[z];
  const int step = gridDim.x * blockDim.x;
  if (vec) {
    const float4* __restrict__ s4 = reinterpret_cast<const float4*>(s);
    float4* __restrict__ d4 = reinterpret_cast<float4*>(d);
#pragma unroll 4
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols / 4; c += step) d4[c] = s4[c];
  } else {
#pragma unroll 4
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += step) d[c] = s[c];
  }
}

int blocks_for(int64_t n, int t) { return (int)std::min<int64_t>((n + t - 1) / t, 148 * 32); }

}  // namespace
}  // namespace apb

using namespace apb;

extern "C" {

int ap_dqn_dueling(const float* z, int64_t ldz, float* q, int64_t ldq, int32_t B, int32_t A, void* stream) {
  if (!z || !q || B < 0 || A < 1) {
    set_error("ap_dqn_dueling: bad arguments");
    return AP_ERR_INVALID;
  }
  if (B == 0) return AP_OK;
  if (A > 256)
    launch_pdl(dueling_wide_kernel, dim3(B), dim3(256), 0, (cudaStream_t)stream, z, ldz, q, ldq, B, A);
  else
    launch_pdl(dueling_kernel, dim3((B + 7) / 8), dim3(256), 0, (cudaStream_t)stream, z, ldz, q, ldq, B, A);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_act(const float* q, int64_t ldq, const uint8_t* mask, int64_t ldm, int32_t E, int32_t A, float epsilon,
               uint64_t seed, int32_t* actions, void* stream) {
  if (!q || !mask || !actions || E < 0 || A < 1) {
    set_error("ap_dqn_act: bad arguments");
    return AP_ERR_INVALID;
  }
  if (E == 0) return AP_OK;
  launch_pdl(act_kernel, dim3((E + 7) / 8), dim3(256), 0, (cudaStream_t)stream, q, ldq, mask, ldm, E, A, epsilon, seed, actions, nullptr,
                                                            0.f, 0.f, 0);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_act_ctl(const float* q, int64_t ldq, const uint8_t* mask, int64_t ldm, int32_t E, int32_t A,
                   float epsilon_start, float epsilon_final, int64_t decay_iters, const int64_t* ctl, int32_t* actions,
                   void* stream) {
  if (!q || !mask || !actions || !ctl || E < 0 || A < 1) {
    set_error("ap_dqn_act_ctl: bad arguments");
    return AP_ERR_INVALID;
  }
  if (E == 0) return AP_OK;
  launch_pdl(act_kernel, dim3((E + 7) / 8), dim3(256), 0, (cudaStream_t)stream, q, ldq, mask, ldm, E, A, 0.f, 0, actions, ctl,
                                                            epsilon_start, epsilon_final, decay_iters);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_td(const float* q, const float* online_next, const float* target_next, int64_t ldq, const int32_t* actions,
              const float* rewards, const uint8_t* done, const uint8_t* next_mask, int64_t ldm, const float* weights,
              int32_t B, int32_t A, float gamma, float huber_delta, float* dz, int64_t ldz, float* td, float* loss,
              void* stream) {
  if (!q || !online_next || !target_next || !actions || !rewards || !done || !next_mask || !weights || !dz || !td ||
      !loss || B < 1 || A < 1) {
    set_error("ap_dqn_td: bad arguments");
    return AP_ERR_INVALID;
  }
  launch_pdl(td_kernel, dim3((B + 7) / 8), dim3(256), 0, (cudaStream_t)stream, q, online_next, target_next, ldq, actions, rewards, done,
                                                           next_mask, ldm, weights, B, A, gamma, huber_delta, dz, ldz,
                                                           td, loss, nullptr, nullptr, 0);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_head_forward(const float* h, int64_t ldh, const float* wh_t, int64_t ldw, const float* bh, int32_t B,
                        int32_t H, int32_t A1, float* q, int64_t ldq, void* stream) {
  if (!h || !wh_t || !bh || !q || B < 0 || H < 1 || A1 < 2) {
    set_error("ap_dqn_head_forward: bad arguments");
    return AP_ERR_INVALID;
  }
  if (A1 > kHeadMax) {
    set_error("ap_dqn_head_forward: head wider than 8 outputs (use the GEMM + ap_dqn_dueling path)");
    return AP_ERR_UNSUPPORTED;
  }
  if (B == 0) return AP_OK;
  const dim3 grid((B + 7) / 8), block(256);
  cudaStream_t s = (cudaStream_t)stream;
  switch (A1) {
    case 2: launch_pdl(head_forward_kernel<2>, dim3(grid), dim3(block), 0, s, h, ldh, wh_t, ldw, bh, B, H, q, ldq); break;
    case 3: launch_pdl(head_forward_kernel<3>, dim3(grid), dim3(block), 0, s, h, ldh, wh_t, ldw, bh, B, H, q, ldq); break;
    case 4: launch_pdl(head_forward_kernel<4>, dim3(grid), dim3(block), 0, s, h, ldh, wh_t, ldw, bh, B, H, q, ldq); break;
    case 5: launch_pdl(head_forward_kernel<5>, dim3(grid), dim3(block), 0, s, h, ldh, wh_t, ldw, bh, B, H, q, ldq); break;
    case 6: launch_pdl(head_forward_kernel<6>, dim3(grid), dim3(block), 0, s, h, ldh, wh_t, ldw, bh, B, H, q, ldq); break;
    case 7: launch_pdl(head_forward_kernel<7>, dim3(grid), dim3(block), 0, s, h, ldh, wh_t, ldw, bh, B, H, q, ldq); break;
    default: launch_pdl(head_forward_kernel<8>, dim3(grid), dim3(block), 0, s, h, ldh, wh_t, ldw, bh, B, H, q, ldq); break;
  }
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_relu_backward_t(float* dh, int64_t lddh, const float* h, int64_t ldh, int32_t B, int32_t H, float* dh_t,
                           int64_t ldt, void* stream) {
  if (!dh || !h || !dh_t || B < 0 || H < 0) {
    set_error("ap_dqn_relu_backward_t: bad arguments");
    return AP_ERR_INVALID;
  }
  const int64_t n = (int64_t)B * H;
  if (n == 0) return AP_OK;
  launch_pdl(relu_bwd_t_kernel, dim3((int)((n + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, dh, lddh, h, ldh, B, H, dh_t, ldt);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_transpose_batch(int32_t n, const float* const* src, const int64_t* ld_src, float* const* dst,
                       const int64_t* ld_dst, const int32_t* rows, const int32_t* cols, void* stream) {
  if (n < 0 || n > 8 || (n > 0 && (!src || !ld_src || !dst || !ld_dst || !rows || !cols))) {
    set_error("ap_transpose_batch: 0..8 segments with host descriptor arrays");
    return AP_ERR_INVALID;
  }
  if (n == 0) return AP_OK;
  TransposeBatch tb{};
  int max_r = 0, max_c = 0;
  for (int i = 0; i < n; ++i) {
    tb.src[i] = src[i];
    tb.dst[i] = dst[i];
    tb.lds[i] = ld_src[i];
    tb.ldd[i] = ld_dst[i];
    tb.rows[i] = rows[i];
    tb.cols[i] = cols[i];
    max_r = std::max(max_r, (int)rows[i]);
    max_c = std::max(max_c, (int)cols[i]);
  }
  const dim3 grid((max_c + 31) / 32, (max_r + 31) / 32, n);
  launch_pdl(transpose_batch_kernel, dim3(grid), dim3(dim3(32, 8)), 0, (cudaStream_t)stream, tb);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_td_ring(const float* q, const float* online_next, const float* target_next, int64_t ldq,
                   const int32_t* indices, const int32_t* ring_actions, const float* ring_rewards,
                   const uint8_t* ring_done, const uint8_t* ring_next_mask, int64_t ldm, const float* weights,
                   int32_t B, int32_t A, float gamma, float huber_delta, float* dz, int64_t ldz, float* dz_t,
                   int64_t ldzt, float* td, float* loss, void* stream) {
  if (!q || !online_next || !target_next || !indices || !ring_actions || !ring_rewards || !ring_done ||
      !ring_next_mask || !weights || !dz || !td || !loss || B < 1 || A < 1) {
    set_error("ap_dqn_td_ring: bad arguments");
    return AP_ERR_INVALID;
  }
  if (A > 64)  // wide action spaces: a CTA per row
    launch_pdl(td_wide_kernel, dim3(B), dim3(256), 0, (cudaStream_t)stream, q, online_next, target_next, ldq, ring_actions, ring_rewards,
                                                        ring_done, ring_next_mask, ldm, weights, B, A, gamma,
                                                        huber_delta, dz, ldz, td, loss, indices, dz_t, ldzt);
  else
    launch_pdl(td_kernel, dim3((B + 7) / 8), dim3(256), 0, (cudaStream_t)stream, q, online_next, target_next, ldq, ring_actions,
                                                             ring_rewards, ring_done, ring_next_mask, ldm, weights, B,
                                                             A, gamma, huber_delta, dz, ldz, td, loss, indices, dz_t,
                                                             ldzt);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_relu_backward(float* dh, const float* h, int64_t n, void* stream) {
  if (n <= 0) return AP_OK;
  launch_pdl(relu_bwd_kernel, dim3(blocks_for(n, 256)), dim3(256), 0, (cudaStream_t)stream, dh, h, n);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_head_backward_dueling(const float* dz, int64_t ldz, const float* wh, int64_t ldw, const float* h,
                                 int64_t ldh, int32_t B, int32_t H, int32_t A1, float* rowsum_scratch, float* dh,
                                 int64_t lddh, float* dh_t, int64_t ldt, void* stream) {
  if (!dz || !wh || !h || !dh || !rowsum_scratch || B < 0 || H < 1 || A1 < 2) {
    set_error("ap_dqn_head_backward_dueling: bad arguments");
    return AP_ERR_INVALID;
  }
  if (B == 0) return AP_OK;
  launch_pdl(head_rowsum_kernel, dim3(H), dim3(256), 0, (cudaStream_t)stream, wh, ldw, A1, rowsum_scratch);
  AP_CUDA_CHECK(cudaGetLastError());
  launch_pdl(head_backward_dueling_kernel, dim3(B), dim3(256), 0, (cudaStream_t)stream, dz, ldz, wh, ldw, h, ldh, rowsum_scratch, H, A1,
                                                                    dh, lddh, dh_t, ldt);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_head_backward(const float* dz, int64_t ldz, const float* wh, int64_t ldw, const float* h, int64_t ldh,
                         int32_t B, int32_t H, int32_t A1, float* dh, int64_t lddh, float* dh_t, int64_t ldt,
                         void* stream) {
  if (!dz || !wh || !h || !dh || B < 0 || H < 1 || A1 < 1) {
    set_error("ap_dqn_head_backward: bad arguments");
    return AP_ERR_INVALID;
  }
  const int64_t n = (int64_t)B * H;
  if (n == 0) return AP_OK;
  if (A1 > 32) {  // wide heads (PP actions): one warp per (row, unit), lanes over the head outputs
    launch_pdl(head_backward_wide_kernel, dim3((int)((n + 7) / 8)), dim3(256), 0, (cudaStream_t)stream, dz, ldz, wh, ldw, h, ldh, B, H,
                                                                                  A1, dh, lddh, dh_t, ldt);
    AP_CUDA_CHECK(cudaGetLastError());
    return AP_OK;
  }
  launch_pdl(head_backward_kernel, dim3((int)((n + 255) / 256)), dim3(256), 0, (cudaStream_t)stream, dz, ldz, wh, ldw, h, ldh, B, H, A1,
                                                                                 dh, lddh, dh_t, ldt);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_colsum(const float* x, int64_t ld, int32_t rows, int32_t cols, float* out, void* stream) {
  if (cols <= 0) return AP_OK;
  launch_pdl(colsum_kernel, dim3((cols + 127) / 128), dim3(128), 0, (cudaStream_t)stream, x, ld, rows, cols, out);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_adam(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1, float beta2,
                float eps, float correct1, float correct2, void* stream) {
  if (n <= 0) return AP_OK;
  launch_pdl(adam_kernel, dim3(blocks_for(n, 256)), dim3(256), 0, (cudaStream_t)stream, params, grads, m, v, n, lr, beta1, beta2, eps,
                                                                     correct1, correct2, nullptr,
             (const float*)nullptr, (int64_t)0);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_adam_ctl_t_adv(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1,
                          float beta2, float eps, const int64_t* ctl, int32_t nseg, const int64_t* seg_off,
                          const int32_t* seg_rows, const int32_t* seg_cols, float* const* seg_dst,
                          const int64_t* seg_ldd, int32_t counter_advanced, void* stream);

int ap_dqn_adam_ctl_t(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1,
                      float beta2, float eps, const int64_t* ctl, int32_t nseg, const int64_t* seg_off,
                      const int32_t* seg_rows, const int32_t* seg_cols, float* const* seg_dst, const int64_t* seg_ldd,
                      void* stream) {
  return ap_dqn_adam_ctl_t_adv(params, grads, m, v, n, lr, beta1, beta2, eps, ctl, nseg, seg_off, seg_rows, seg_cols,
                               seg_dst, seg_ldd, 0, stream);
}

int ap_dqn_adam_ctl_t_adv(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1,
                          float beta2, float eps, const int64_t* ctl, int32_t nseg, const int64_t* seg_off,
                          const int32_t* seg_rows, const int32_t* seg_cols, float* const* seg_dst,
                          const int64_t* seg_ldd, int32_t counter_advanced, void* stream) {
  if (!ctl || nseg < 0 || nseg > 8 || (nseg > 0 && (!seg_off || !seg_rows || !seg_cols || !seg_dst || !seg_ldd))) {
    set_error("ap_dqn_adam_ctl_t: bad arguments (0..8 segments, host descriptor arrays)");
    return AP_ERR_INVALID;
  }
  if (n <= 0) return AP_OK;
  AdamSegments segs{};
  segs.n = nseg;
  segs.t_add = counter_advanced ? 0 : 1;
  for (int s = 0; s < nseg; ++s) {
    segs.off[s] = seg_off[s];
    segs.rows[s] = seg_rows[s];
    segs.cols[s] = seg_cols[s];
    segs.dst[s] = seg_dst[s];
    segs.ldd[s] = seg_ldd[s];
  }
  // tiled path when the segments are disjoint and inside [0, n)
  int order[8];
  for (int s = 0; s < nseg; ++s) order[s] = s;
  std::sort(order, order + nseg, [&](int a, int b) { return segs.off[a] < segs.off[b]; });
  bool tiled = std::getenv("AP_ADAM_FLAT") == nullptr;
  int64_t end = 0;
  for (int k = 0; k < nseg && tiled; ++k) {
    const int s = order[k];
    tiled = segs.off[s] >= end && segs.rows[s] > 0 && segs.cols[s] > 0;
    end = segs.off[s] + (int64_t)segs.rows[s] * segs.cols[s];
  }
  tiled = tiled && end <= n;
  if (tiled) {
    AdamTiles at{};
    at.segs = segs;
    at.tile_base[0] = 0;
    for (int s = 0; s < nseg; ++s) {
      at.tcols[s] = (segs.cols[s] + 31) / 32;
      at.tile_base[s + 1] = at.tile_base[s] + (int64_t)((segs.rows[s] + 31) / 32) * at.tcols[s];
    }
    int64_t lo = 0;
    at.ngap = 0;
    at.gap_base[0] = 0;
    for (int k = 0; k <= nseg; ++k) {
      const int64_t hi = k < nseg ? segs.off[order[k]] : n;
      if (hi > lo) {
        at.gap_lo[at.ngap] = lo;
        at.gap_base[at.ngap + 1] = at.gap_base[at.ngap] + (hi - lo);
        ++at.ngap;
      }
      if (k < nseg) lo = segs.off[order[k]] + (int64_t)segs.rows[order[k]] * segs.cols[order[k]];
    }
    const int64_t blocks = at.tile_base[nseg] + (at.gap_base[at.ngap] + 255) / 256;
    launch_pdl(adam_tile_kernel, dim3((unsigned)blocks), dim3(256), 0, (cudaStream_t)stream, params, grads, m, v, lr, beta1, beta2, eps,
                                                                         ctl, at);
  } else {
    launch_pdl(adam_t_kernel, dim3(blocks_for(n, 256)), dim3(256), 0, (cudaStream_t)stream, params, grads, m, v, n, lr, beta1, beta2, eps,
                                                                         ctl, segs);
  }
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_adam_ctl(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1,
                    float beta2, float eps, const int64_t* ctl, void* stream) {
  if (!ctl) {
    set_error("ap_dqn_adam_ctl: null control block");
    return AP_ERR_INVALID;
  }
  if (n <= 0) return AP_OK;
  launch_pdl(adam_kernel, dim3(blocks_for(n, 256)), dim3(256), 0, (cudaStream_t)stream, params, grads, m, v, n, lr, beta1, beta2, eps,
                                                                     1.f, 1.f, ctl, (const float*)nullptr,
             (int64_t)0);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_per_sample(const double* priorities, int32_t n, double alpha, double beta, const double* uniforms, int32_t B,
                  double* scratch, int32_t* indices, float* weights, void* stream) {
  if (!priorities || !uniforms || !scratch || !indices || !weights || n < 1 || B < 1) {
    set_error("ap_per_sample: bad arguments");
    return AP_ERR_INVALID;
  }
  // scratch: [n] scaled + [n + B] cdf / weights
  launch_pdl(per_sample_kernel, dim3(1), dim3(512), 0, (cudaStream_t)stream, priorities, n, alpha, beta, uniforms, B, scratch,
                                                         scratch + n, indices, weights, (const int64_t*)nullptr);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_dqn_adam_tab(float* params, const float* grads, float* m, float* v, int64_t n, float lr, float beta1,
                    float beta2, float eps, const float* ctab, const int64_t* ctl, int64_t t_offset, void* stream) {
  if (!ctab || !ctl) {
    set_error("ap_dqn_adam_tab: null table or control block");
    return AP_ERR_INVALID;
  }
  if (n <= 0) return AP_OK;
  launch_pdl(adam_kernel, dim3(blocks_for(n, 256)), dim3(256), 0, (cudaStream_t)stream, params, grads, m, v, n, lr,
             beta1, beta2, eps, 1.f, 1.f, (const int64_t*)ctl, ctab, t_offset);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_per_update(double* priorities, const int32_t* indices, const float* td, int32_t B, void* stream) {
  if (B <= 0) return AP_OK;
  launch_pdl(per_update_kernel, dim3((B + 127) / 128), dim3(128), 0, (cudaStream_t)stream, priorities, indices, td, B);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_gather_rows_pair(const float* src0, int64_t lds0, float* dst0, int64_t ldd0, const float* src1, int64_t lds1,
                        float* dst1, int64_t ldd1, const int32_t* idx, int32_t B, int32_t cols, void* stream) {
  if (B <= 0 || cols <= 0) return AP_OK;
  if (B > 65535 || !src0 || !dst0 || !idx) {
    set_error("ap_gather_rows: bad arguments (at most 65535 rows per call)");
    return AP_ERR_INVALID;
  }
  const int pairs = src1 ? 2 : 1;
  GatherPair gp{{src0, src1}, {lds0, lds1}, {dst0, dst1}, {ldd0, ldd1}};
  uintptr_t bases = reinterpret_cast<uintptr_t>(src0) | reinterpret_cast<uintptr_t>(dst0);
  int64_t strides = lds0 | ldd0;
  if (src1) {
    bases |= reinterpret_cast<uintptr_t>(src1) | reinterpret_cast<uintptr_t>(dst1);
    strides |= lds1 | ldd1;
  }
  const int vec = cols % 4 == 0 && strides % 4 == 0 && (bases & 15) == 0;
  const int per_row = vec ? cols / 4 : cols;
  const dim3 grid((unsigned)std::max(1, std::min((per_row + 255) / 256, 16)), (unsigned)B, (unsigned)pairs);
  launch_pdl(gather_rows_kernel, grid, dim3(256), 0, (cudaStream_t)stream, gp, idx, B, cols, vec);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

int ap_gather_rows(const float* src, int64_t lds, const int32_t* idx, int32_t B, int32_t cols, float* dst,
                   int64_t ldd, void* stream) {
  return ap_gather_rows_pair(src, lds, dst, ldd, nullptr, 0, nullptr, 0, idx, B, cols, stream);
}

}  // extern "C"
