// peak.cu -- FP64 peak probes for the roofline denominators.
// MEASURED_PEAKS.json carries HBM and bf16 only; bench.py runs these once per process.
//   qtt_probe_dfma : 8 independent DFMA chains per thread  (2 flops / FMA)
//   qtt_probe_dmma : 4 independent mma.sync m8n8k4 f64 chains per warp (512 flops / MMA)
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(256) k_dfma(double *out, int iters) {
  double a[8];
  const double x = 1.0 + 1e-9 * threadIdx.x, y = 0.999999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], y, x);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678) out[blockIdx.x] = s;   // practically never: keeps the chain alive
}

__global__ void __launch_bounds__(256) k_dmma(double *out, int iters) {
  double c[4][2];
  const double av = 1.0 + 1e-9 * threadIdx.x, bv = 0.5;
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(av), "d"(bv));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[blockIdx.x] = s;
}

extern "C" {
// flops executed by one launch: dfma: blocks*256*iters*16*8*2 ; dmma: blocks*8*iters*8*4*512
int qtt_probe_dfma(double *out, int blocks, int iters, void *stream) {
  k_dfma<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, iters);
  return (int)cudaGetLastError();
}
int qtt_probe_dmma(double *out, int blocks, int iters, void *stream) {
  k_dmma<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, iters);
  return (int)cudaGetLastError();
}
}
