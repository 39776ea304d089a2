// numpy Generator samplers on the device (host-callable too, for the CPU tests):
// Generator.normal (ziggurat, distributions.c random_standard_normal with the
// tables of np_ziggurat.h) and Generator.binomial (random_binomial: BTPE for
// n * min(p, 1-p) > 30, Kachitvichyanukul & Schmeiser's algorithm as numpy
// writes it).  Both consume a data-dependent number of PCG64 outputs, so a
// stream is sampled sequentially by one thread.  The reference draws its
// synthetic PP-infer profiles through these (reference dataproc.py:123-145:
// N(0.5, 0.15) clipped to [0, 1]; B(100, 0.5) / 100).
// Compiled with -fmad=false: every product and sum rounds separately, as numpy's
// baseline-x86-64 build does.
#pragma once

#include <cmath>
#include <cstdint>

#include "np_ziggurat.h"
#include "pcg64.cuh"

namespace apb {

constexpr double kZigNorR = 3.6541528853610088;       // ziggurat_nor_r
constexpr double kZigNorInvR = 0.27366123732975828;   // ziggurat_nor_inv_r

__host__ __device__ inline double np_standard_normal(NpPcg64& g) {
  for (;;) {
    uint64_t r = g.next64();
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 0x1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * np_wi_double[idx];
    if (sign & 0x1) x = -x;
    if (rabs < np_ki_double[idx]) return x;  // 99.3% of the draws
    if (idx == 0) {
      for (;;) {
        // 1.0 - U avoids log(0.0) (numpy GH 13361)
        const double xx = -kZigNorInvR * log1p(-g.next_double());
        const double yy = -log1p(-g.next_double());
        if (yy + yy > xx * xx) return ((rabs >> 8) & 0x1) ? -(kZigNorR + xx) : kZigNorR + xx;
      }
    } else {
      if (((np_fi_double[idx - 1] - np_fi_double[idx]) * g.next_double() + np_fi_double[idx]) < exp(-0.5 * x * x))
        return x;
    }
  }
}

// random_binomial_btpe (numpy distributions.c); the per-(n, p) setup of binomial_t is
// recomputed, which yields the same values numpy caches.  Kept out of line: inlined into
// the per-environment loop, ptxas -O3 miscompiles it for divergent warps (wrong draws for
// every thread once lanes take different rejection paths; -O0, -G and a call are exact).
__host__ __device__ __noinline__ int64_t np_binomial_btpe(NpPcg64& g, int64_t n, double p) {
  const double r = fmin(p, 1.0 - p);
  const double q = 1.0 - r;
  const double fm = n * r + r;
  const int64_t m = (int64_t)floor(fm);
  const double p1 = floor(2.195 * sqrt(n * r * q) - 4.6 * q) + 0.5;
  const double xm = m + 0.5;
  const double xl = xm - p1;
  const double xr = xm + p1;
  const double c = 0.134 + 20.5 / (15.3 + m);
  double a = (fm - xl) / (fm - xl * r);
  const double laml = a * (1.0 + a / 2.0);
  a = (xr - fm) / (xr * q);
  const double lamr = a * (1.0 + a / 2.0);
  const double p2 = p1 * (1.0 + 2.0 * c);
  const double p3 = p2 + c / laml;
  const double p4 = p3 + c / lamr;
  const double nrq = n * r * q;
  int64_t y;
  for (;;) {  // Step10
    double u = g.next_double() * p4;
    double v = g.next_double();
    if (u <= p1) {
      y = (int64_t)floor(xm - p1 * v + u);
      break;  // Step60
    }
    if (u <= p2) {  // Step20
      const double x = xl + (u - p1) / c;
      v = v * c + 1.0 - fabs(m - x + 0.5) / p1;
      if (v > 1.0) continue;
      y = (int64_t)floor(x);
    } else if (u <= p3) {  // Step30
      y = (int64_t)floor(xl + log(v) / laml);
      if ((y < 0) || (v == 0.0)) continue;
      v = v * (u - p2) * laml;
    } else {  // Step40
      y = (int64_t)floor(xr - log(v) / lamr);
      if ((y > n) || (v == 0.0)) continue;
      v = v * (u - p3) * lamr;
    }
    // Step50
    const int64_t k = y > m ? y - m : m - y;
    if ((k > 20) && (k < ((nrq) / 2.0 - 1))) {
      // Step52
      const double kd = (double)k;
      const double rho = (kd / (nrq)) * ((kd * (kd / 3.0 + 0.625) + 0.16666666666666666) / nrq + 0.5);
      const double t = -kd * kd / (2 * nrq);
      const double A = log(v);
      if (A < (t - rho)) break;
      if (A > (t + rho)) continue;
      const double x1 = y + 1, f1 = m + 1, z = n + 1 - m, w = n - y + 1;
      const double x2 = x1 * x1, f2 = f1 * f1, z2 = z * z, w2 = w * w;
      if (A > (xm * log(f1 / x1) + (n - m + 0.5) * log(z / w) + (y - m) * log(w * r / (x1 * q)) +
               (13680. - (462. - (132. - (99. - 140. / f2) / f2) / f2) / f2) / f1 / 166320. +
               (13680. - (462. - (132. - (99. - 140. / z2) / z2) / z2) / z2) / z / 166320. +
               (13680. - (462. - (132. - (99. - 140. / x2) / x2) / x2) / x2) / x1 / 166320. +
               (13680. - (462. - (132. - (99. - 140. / w2) / w2) / w2) / w2) / w / 166320.))
        continue;
      break;
    }
    const double s = r / q;
    const double aa = s * (n + 1);
    double F = 1.0;
    if (m < y) {
      for (int64_t i = m + 1; i <= y; i++) F *= (aa / i - s);
    } else if (m > y) {
      for (int64_t i = y + 1; i <= m; i++) F /= (aa / i - s);
    }
    if (v > F) continue;
    break;
  }
  if (p > 0.5) y = n - y;  // Step60
  return y;
}

// Generator.binomial(n, p) for the BTPE regime (n * min(p, 1 - p) > 30)
__host__ __device__ inline int64_t np_binomial(NpPcg64& g, int64_t n, double p) {
  if (n == 0 || p == 0.0) return 0;
  if (p <= 0.5) return np_binomial_btpe(g, n, p);
  return n - np_binomial_btpe(g, n, 1.0 - p);
}

}  // namespace apb
