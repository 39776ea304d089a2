// Prioritized-replay sampling in numpy's exact arithmetic, one CTA (agent.py:207-223):
//
//   scaled = priorities[:n] ** alpha
//   probs  = scaled / scaled.sum()                  (numpy pairwise summation)
//   idx    = rng.choice(n, B, p=probs)              (cdf = probs.cumsum(); cdf /= cdf[-1];
//                                                    searchsorted(uniforms, side='right'))
//   w      = (n * probs[idx]) ** -beta;  w /= w.max()
//
// Everything but the cumsum runs across the CTA.  numpy's pairwise sum is a fixed binary
// recursion over blocks of <= 128 elements (PW_BLOCKSIZE): thread 0 lists the blocks, the
// block sums run in parallel (8 interleaved accumulators each, numpy's unrolled loop), and
// thread 0 adds them back up in the recursion's order.  The cumsum is numpy's sequential
// chain of adds on one thread, its operands prefetched 16 at a time.
#pragma once

#include <cstdint>

#ifndef ST
#define ST(k) \
  do {        \
  } while (0)
#endif

namespace apb {
namespace {  // internal linkage: included by several translation units

constexpr int kPerMaxNodes = 1024;  // nodes of the pairwise recursion handled in parallel (24 KB)

// numpy pairwise summation of one block of <= 128 doubles
// (numpy/_core/src/umath/loops_utils.h.src)
__device__ __forceinline__ double np_pairwise_leaf(const double* x, int64_t m) {
  if (m < 8) {
    double v = -0.0;  // numpy starts from -0.0 to preserve -0.0 sums
    for (int64_t i = 0; i < m; ++i) v += x[i];
    return v;
  }
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = x[k];
  int64_t i;
  for (i = 8; i < m - (m % 8); i += 8)
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] += x[i + k];
  double v = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < m; ++i) v += x[i];
  return v;
}

// Walk of the recursion sum(a, n) = sum(a, n2) + sum(a + n2, n - n2), n2 = n/2 rounded down to
// a multiple of 8, with an explicit post-order stack.  LEAF(off, len) gives a block's sum.
template <typename Leaf>
__device__ double np_pairwise_walk(int64_t n, Leaf leaf) {
  struct Frame {
    int64_t off, n;
    int state;
    double left;
  };
  Frame fr[64];
  int top = 0;
  fr[0] = {0, n, 0, 0.0};
  double ret = 0.0;
  while (top >= 0) {
    Frame& f = fr[top];
    if (f.n <= 128) {
      ret = leaf(f.off, f.n);
      --top;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      fr[top + 1] = {f.off, n2, 0, 0.0};
      ++top;
    } else if (f.state == 1) {
      f.left = ret;
      f.state = 2;
      fr[top + 1] = {f.off + n2, f.n - n2, 0, 0.0};
      ++top;
    } else {
      ret = f.left + ret;
      --top;
    }
  }
  return ret;
}

struct PerShared {
  int64_t node_off[kPerMaxNodes];
  int32_t node_len[kPerMaxNodes];
  int32_t node_child[kPerMaxNodes];  // left child (right = left + 1), -1 a block, -2 summed serially
  double node_sum[kPerMaxNodes];
  uint8_t node_depth[kPerMaxNodes];
  int nnodes, max_depth;
  double total, last, wmax;
  double wred[32];
};

// The recursion's nodes for n elements, breadth first (children after their parent).  One thread.
__device__ __forceinline__ void per_tree(int n, PerShared& S) {
  int cnt = 1, dmax = 0;
  S.node_off[0] = 0, S.node_len[0] = n, S.node_depth[0] = 0;
  for (int i = 0; i < cnt; ++i) {
    const int len = S.node_len[i];
    if (len <= 128 || cnt + 2 > kPerMaxNodes) {
      S.node_child[i] = len <= 128 ? -1 : -2;
      continue;
    }
    int n2 = len / 2;
    n2 -= n2 % 8;
    const int d = S.node_depth[i] + 1;
    dmax = d > dmax ? d : dmax;
    S.node_child[i] = cnt;
    S.node_off[cnt] = S.node_off[i], S.node_len[cnt] = n2, S.node_depth[cnt] = (uint8_t)d;
    S.node_off[cnt + 1] = S.node_off[i] + n2, S.node_len[cnt + 1] = len - n2, S.node_depth[cnt + 1] = (uint8_t)d;
    cnt += 2;
  }
  S.nnodes = cnt;
  S.max_depth = dmax;
}

// a subtree past the node table's capacity, summed serially (out of line: its stack of
// recursion frames stays out of the common path)
__device__ __noinline__ double np_pairwise_serial(const double* x, int64_t n) {
  return np_pairwise_walk(n, [&](int64_t off, int64_t len) { return np_pairwise_leaf(x + off, len); });
}

// total = numpy's pairwise sum of scaled[0, n) over the tree of per_tree (every thread; the
// block sums in parallel, then the internal nodes level by level).  Ends with a barrier.
__device__ __forceinline__ void per_total(const double* scaled, PerShared& S) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nn = S.nnodes;
  // Blocks of >= 8 elements: 8 lanes per block, lane k runs numpy's accumulator r[k] (x[k],
  // x[k + 8], ... in order), then the fixed tree ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7))
  // over shuffles and the m % 8 tail on lane 0.  (Block offsets are multiples of 8, so one lane
  // per block would put every lane's loads on the same two banks.)
  const int grp = tid >> 3, k = tid & 7, ngrp = nt >> 3;
  for (int i0 = 0; i0 < nn; i0 += ngrp) {
    const int i = i0 + grp;
    const int c = i < nn ? S.node_child[i] : 0;
    const int m = c == -1 ? S.node_len[i] : 0;
    const bool big = c == -1 && m >= 8;
    double r = 0.0;
    const double* x = big ? scaled + S.node_off[i] : nullptr;
    const int m8 = m - (m % 8);
    if (big) {
      r = x[k];
      for (int j = 8 + k; j < m8; j += 8) r += x[j];
    }
    // the tree over the 8 lanes of the group (every lane of the warp takes part in the shuffles)
    const double r1 = __shfl_xor_sync(0xffffffffu, r, 1);
    const double p01 = (k & 1) ? r1 + r : r + r1;  // lanes 2q hold r[2q] + r[2q + 1]
    const double p23 = __shfl_xor_sync(0xffffffffu, p01, 2);
    const double q = (k & 2) ? p23 + p01 : p01 + p23;  // lanes 0, 4: (r0 + r1) + (r2 + r3), (r4 + r5) + (r6 + r7)
    const double q4 = __shfl_xor_sync(0xffffffffu, q, 4);
    if (big && k == 0) {
      double v = q + q4;
      for (int j = m8; j < m; ++j) v += x[j];
      S.node_sum[i] = v;
    }
    if (i < nn && k == 0) {
      if (c == -1 && m < 8)
        S.node_sum[i] = np_pairwise_leaf(scaled + S.node_off[i], m);
      else if (c == -2)
        S.node_sum[i] = np_pairwise_serial(scaled + S.node_off[i], S.node_len[i]);
    }
  }
  __syncthreads();
  ST(4);
  // internal nodes level by level, deepest first (one thread per node; ~log2(n / 64) levels)
  for (int d = S.max_depth - 1; d >= 0; --d) {
    for (int i = tid; i < nn; i += nt) {
      const int c = S.node_child[i];
      if (c >= 0 && S.node_depth[i] == d) S.node_sum[i] = S.node_sum[c] + S.node_sum[c + 1];
    }
    __syncthreads();
  }
  if (tid == 0) S.total = S.node_sum[0];
  __syncthreads();
}

// From scaled[0, n) and S.total: probs, numpy's cdf (sequential cumsum), the B searchsorted
// draws and the normalised importance weights, in two calls (every thread).  probs: n + B
// doubles.  The cumsum overwrites scaled (p = probs[i] is all the weights need afterwards).
// (1) probs and the cdf chain: every thread divides, then thread 0 runs the chain while the
// others are free (the caller syncs before per_pick)
__device__ __forceinline__ void per_cdf(double* __restrict__ scaled, int n, double* __restrict__ probs,
                                        PerShared& S) {
  const int tid = threadIdx.x, nt = blockDim.x;
  // probs = scaled / total (independent divisions)
  const double total = S.total;
  for (int i = tid; i < n; i += nt) probs[i] = scaled[i] / total;
  __syncthreads();
  ST(6);
  if (tid == 0) {
    // cdf = probs.cumsum(): one chain of adds, the critical path; operands 16 ahead in registers
    double* __restrict__ cdf = scaled;
    double acc = probs[0];
    cdf[0] = acc;
    int i = 1;
    for (; i + 16 <= n; i += 16) {
      double x[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) x[k] = probs[i + k];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        acc = acc + x[k];
        cdf[i + k] = acc;
      }
    }
    for (; i < n; ++i) {
      acc = acc + probs[i];
      cdf[i] = acc;
    }
    S.last = acc;
  }
}

// (2) after a barrier: searchsorted on cdf / cdf[-1] and the normalised importance weights
__device__ __forceinline__ void per_pick(const double* __restrict__ scaled, int n, double beta, const double* u,
                                         int B, double* __restrict__ probs, int32_t* __restrict__ idx_out,
                                         float* __restrict__ w_out, PerShared& S) {
  const int tid = threadIdx.x, nt = blockDim.x;
  ST(7);
  // cdf /= cdf[-1]; searchsorted(side='right'): the first i with cdf[i] / last > u, each
  // probe's quotient computed where it is needed (the same rounded value)
  const double* cdf = scaled;
  const double last = S.last;
  double wloc = 0.0;
  for (int b = tid; b < B; b += nt) {
    const double ub = u[b];
    // fl(c / last) <= u is decided by c against u * last with a 2^-48 relative margin (far wider
    // than the 2^-53 rounding of either side); only a c inside the margin pays the division
    const double ul = ub * last, mg = ul * 0x1p-48, lo_t = ul - mg, hi_t = ul + mg;
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      const double c = cdf[mid];
      const bool le = c <= lo_t ? true : (c >= hi_t ? false : c / last <= ub);
      if (le)
        lo = mid + 1;
      else
        hi = mid;
    }
    idx_out[b] = lo;
    const double w = pow((double)n * probs[lo], -beta);
    probs[n + b] = w;
    wloc = fmax(wloc, w);
  }
  for (int o = 16; o; o >>= 1) wloc = fmax(wloc, __shfl_xor_sync(0xffffffffu, wloc, o));
  if ((tid & 31) == 0) S.wred[tid >> 5] = wloc;
  __syncthreads();
  if (tid < 32) {
    double m = tid < (nt >> 5) ? S.wred[tid] : 0.0;
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (tid == 0) S.wmax = m;
  }
  __syncthreads();
  for (int b = tid; b < B; b += nt) w_out[b] = (float)(probs[n + b] / S.wmax);
}

// The whole sample with scaled = priorities ** alpha computed here (every thread).
__device__ __noinline__ void per_sample_block(const double* __restrict__ prio, int n, double alpha, double beta,
                                              const double* u, int B, double* scaled, double* cdf,
                                              int32_t* __restrict__ idx_out, float* __restrict__ w_out,
                                              PerShared& S) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) scaled[i] = pow(prio[i], alpha);
  if (threadIdx.x == 0) per_tree(n, S);
  __syncthreads();
  per_total(scaled, S);
  per_cdf(scaled, n, cdf, S);  // (cdf: n + B doubles)
  __syncthreads();
  per_pick(scaled, n, beta, u, B, cdf, idx_out, w_out, S);
}

}  // namespace
}  // namespace apb
