// cs_probe.cuh -- FP64 pipe peak probe (MEASURED_PEAKS.json has no FP64
// entry): independent DFMA chains, 8 per thread, no memory traffic.
#pragma once
#include "cs_common.cuh"

__global__ void __launch_bounds__(256) k_dfma_probe(int iters, double seed, double *out) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = __fma_rn(a0, m, c); a1 = __fma_rn(a1, m, c); a2 = __fma_rn(a2, m, c);
      a3 = __fma_rn(a3, m, c); a4 = __fma_rn(a4, m, c); a5 = __fma_rn(a5, m, c);
      a6 = __fma_rn(a6, m, c); a7 = __fma_rn(a7, m, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

// flops per launch = blocks * 256 * iters * 16 * 8 * 2
extern "C" int cs_probe_dfma(int blocks, int iters, double *out, void *stream) {
  k_dfma_probe<<<blocks, 256, 0, cs_stream(stream)>>>(iters, 1.0, out);
  return cs_check_launch("probe_dfma");
}
