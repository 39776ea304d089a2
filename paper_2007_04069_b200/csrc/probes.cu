// Measurement probes for roofline denominators that MEASURED_PEAKS.json lacks
// (the PP-train cost kernels are bound by fp64 add throughput).
//
// ap_probe_fp64_add: every thread runs 8 independent fp64 add chains for
// `iters` iterations, so the FP64 pipe, not add latency, is the limit.  The
// caller times the launch and divides grid*block*8*iters adds by it.
#include "engine.h"

namespace apb {
namespace {

__global__ void __launch_bounds__(256) fp64_add_probe(int64_t iters, double step, double* out) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int64_t k = 0; k < iters; ++k) {
    a0 += step;
    a1 += step;
    a2 += step;
    a3 += step;
    a4 += step;
    a5 += step;
    a6 += step;
    a7 += step;
  }
  const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (s == -1.0) out[0] = s;  // never true: keeps the chains live
}

}  // namespace
}  // namespace apb

using namespace apb;

extern "C" {

int ap_probe_fp64_add(int32_t blocks, int64_t iters, double* scratch_dev, void* stream) {
  if (blocks < 1 || iters < 1 || !scratch_dev) {
    set_error("ap_probe_fp64_add: bad arguments");
    return AP_ERR_INVALID;
  }
  fp64_add_probe<<<blocks, 256, 0, (cudaStream_t)stream>>>(iters, 1e-300, scratch_dev);
  AP_CUDA_CHECK(cudaGetLastError());
  return AP_OK;
}

}  // extern "C"
