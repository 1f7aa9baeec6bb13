// lat.cu -- micro-probes used to size the FP64 latency chains of the Jacobi / QR kernels:
// dependent-chain latency (cycles) of DFMA, 64-bit SHFL, MUFU rsqrt/rcp (f64 approx), LDS,
// and the raw relative error of rsqrt.approx.f64 / rcp.approx.f64 (how many Newton steps
// the rotation parameters need).  Diagnostics only; not on the product path.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ double rsq_approx(double x) {
  double y;
  asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rcp_approx(double x) {
  double y;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// out[0..5]: cycles per dependent op for dfma, shfl64, rsqrt-approx, rcp-approx, lds64, dadd
__global__ void k_lat(double *out, double seed, int iters) {
  __shared__ double sm[64];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 64) sm[threadIdx.x] = (double)threadIdx.x;
  __syncthreads();
  double x = seed + lane * 1e-3;
  long long t0, t1;
  // DFMA
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-9);
  t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
  // SHFL 64
  double y = x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) y = __shfl_xor_sync(0xffffffffu, y, 1);
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (double)(t1 - t0) / iters;
  // rsqrt approx
  double z = 1.5 + x * 1e-12;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) z = rsq_approx(z);
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (double)(t1 - t0) / iters;
  // rcp approx
  double w = 1.5 + x * 1e-12;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) w = rcp_approx(w);
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (double)(t1 - t0) / iters;
  // LDS 64 (pointer chase through values)
  int idx = lane & 7;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = (int)sm[idx] & 31;
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (double)(t1 - t0) / iters;
  // DADD
  double v = x;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) v = v + 1e-9;
  t1 = clock64();
  if (threadIdx.x == 0) out[5] = (double)(t1 - t0) / iters;
  if (threadIdx.x == 0) out[6] = x + y + z + w + idx + v;   // keep results live
}

// max relative error of the raw approximations over n log-uniform inputs in [2^-40, 2^40]
__global__ void k_approx_err(double *out, int n) {
  double er = 0.0, ec = 0.0;
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x) {
    const double e = -40.0 + 80.0 * ((double)i + 0.5) / n;
    const double x = exp2(e) * (1.0 + 0.37 * sin((double)i));
    const double r = rsq_approx(x), c = rcp_approx(x);
    er = fmax(er, fabs(r * sqrt(x) - 1.0));
    ec = fmax(ec, fabs(c * x - 1.0));
  }
  for (int o = 16; o > 0; o >>= 1) {
    er = fmax(er, __shfl_xor_sync(0xffffffffu, er, o));
    ec = fmax(ec, __shfl_xor_sync(0xffffffffu, ec, o));
  }
  if ((threadIdx.x & 31) == 0) {
    unsigned long long *o = (unsigned long long *)out;
    atomicMax(o + 0, (unsigned long long)__double_as_longlong(er));   // non-negative doubles order as ints
    atomicMax(o + 1, (unsigned long long)__double_as_longlong(ec));
  }
}

extern "C" int qtt_probe_latency(double *out, int iters, void *stream) {
  k_lat<<<1, 32, 0, (cudaStream_t)stream>>>(out, 1.25, iters);
  cudaMemsetAsync(out + 8, 0, 2 * sizeof(double), (cudaStream_t)stream);
  k_approx_err<<<64, 256, 0, (cudaStream_t)stream>>>(out + 8, 1 << 22);
  return (int)cudaGetLastError();
}

// Throughput probes: 8 warps (one CTA per SM, grid = #SMs), each issuing independent
// 32-bit SHFL (8 chains) or broadcast LDS.64 (8 chains); out[0] = cycles per SHFL per SM,
// out[1] = cycles per LDS per SM (SM-wide: total instructions issued by the 8 warps).
__global__ void __launch_bounds__(256, 1) k_tput(double *out, int iters) {
  __shared__ double sm[256];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  int r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = threadIdx.x + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = __shfl_xor_sync(0xffffffffu, r[i], 1 + (i & 3));
  }
  __syncthreads();
  long long t1 = clock64();
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  const int base = (threadIdx.x >> 5) * 8;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] += sm[(base + i + it) & 255];
  }
  __syncthreads();
  long long t2 = clock64();
  int s = 0;
  double a = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { s += r[i]; a += acc[i]; }
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    out[0] = (double)(t1 - t0) / (iters * 8.0 * 8.0);
    out[1] = (double)(t2 - t1) / (iters * 8.0 * 8.0);
    out[2] = s + a;
  }
}

extern "C" int qtt_probe_tput(double *out, int iters, int blocks, void *stream) {
  k_tput<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, iters);
  return (int)cudaGetLastError();
}

// accuracy of the one-step Halley rsqrt used by the rotation parameters (common.cuh)
__global__ void k_rsqrt_err(double *out, int n) {
  double er = 0.0;
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i < n; i += blockDim.x * gridDim.x) {
    const double e = -40.0 + 80.0 * ((double)i + 0.5) / n;
    const double x = exp2(e) * (1.0 + 0.37 * sin((double)i));
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double h = x * y, ee = fma(-h, y, 1.0), t = fma(0.375, ee, 0.5), ye = y * ee;
    y = fma(ye, t, y);
    er = fmax(er, fabs(y * sqrt(x) - 1.0));
  }
  for (int o = 16; o > 0; o >>= 1) er = fmax(er, __shfl_xor_sync(0xffffffffu, er, o));
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long *)out, (unsigned long long)__double_as_longlong(er));
}

extern "C" int qtt_probe_rsqrt_err(double *out, void *stream) {
  cudaMemsetAsync(out, 0, sizeof(double), (cudaStream_t)stream);
  k_rsqrt_err<<<64, 256, 0, (cudaStream_t)stream>>>(out, 1 << 22);
  return (int)cudaGetLastError();
}
