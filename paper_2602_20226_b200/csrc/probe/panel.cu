__device__ long long g_blktrace[8 * 16];
#define QTT_BLK_TRACE g_blktrace
// panel.cu -- micro-probe of the small path's a3 (qr_small.cuh): cycles of one 8-column register
// panel factorisation (qr_panel) with the other warps idle, and of a whole qr_of_TH on a 128 x 256
// site matrix.  Diagnostics only; not on the product path.
#include <cuda_runtime.h>
#include "../qr_small.cuh"

using namespace qtt;

__global__ void __launch_bounds__(kST, 1) k_panel_probe(const double *T, long long *out, int mode, int reps) {
  extern __shared__ double sm[];
  double *Rp = sm, *Bk = Rp + kRpDoubles, *Ysm = Bk + kQBkDoubles, *tau = Ysm + 16 * kYld;
  const int warp = threadIdx.x >> 5;
  const int m = 128, n = 256;
  if (mode == 0) {
    for (int i = threadIdx.x; i < kRpDoubles; i += kST) Rp[i] = 0.0;
    for (int idx = threadIdx.x; idx < kSmall * m; idx += kST) {
      const int j = idx / kSmall, i = idx % kSmall;
      Bk[i * kLdQ + j] = T[(size_t)j * n + i];
    }
    __syncthreads();
    if (warp == kSW - 1) {
      const long long t0 = clock64();
      for (int r = 0; r < reps; ++r)
        for (int j0 = 0; j0 < m; j0 += kPanel) qr_panel(Rp, Bk, tau, m, j0);
      const long long t1 = clock64();
      if ((threadIdx.x & 31) == 0) out[0] = (t1 - t0) / reps;
    }
  } else {
    __syncthreads();
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) qr_of_TH(T, m, n, Rp, Bk, tau, Ysm);
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / reps;
  }
}

extern "C" int qtt_probe_panel(const double *T_dev, long long *cycles_host, int mode, int reps) {
  long long *d;
  cudaMalloc(&d, sizeof(long long));
  const size_t smem = (size_t)(kRpDoubles + kQBkDoubles + 16 * kYld + kSmall) * sizeof(double);
  cudaFuncSetAttribute(k_panel_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_panel_probe<<<1, kST, smem>>>(T_dev, d, mode, reps);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(cycles_host, d, sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}

// a1 site (orth.cuh orth_site_reg<4, 8>) on a 64 x 128 core (M^T 128 x 64) with a 128 x 64 left
// neighbour: cycles of one call (fresh inputs each repetition)
#include "../orth.cuh"
__global__ void __launch_bounds__(kThreads, 1) k_orth_probe(const double *core0, const double *prev0, double *core,
                                                            double *prev, long long *out, int reps) {
  extern __shared__ double sm[];
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < 64 * 128; i += kThreads) { core[i] = core0[i]; prev[i] = prev0[i]; }
    __syncthreads();
    const long long t0 = clock64();
    orth_site_reg<4, 8>(core, 128, 64, prev, 128, sm);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) out[0] = tot / reps;
}

extern "C" int qtt_probe_orth(const double *core0, const double *prev0, double *core, double *prev,
                              long long *cycles_host, int reps) {
  long long *d;
  cudaMalloc(&d, sizeof(long long));
  const size_t smem = (size_t)orth_reg_smem(4, 128, 64, 128) * sizeof(double);
  cudaFuncSetAttribute(k_orth_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_orth_probe<<<1, kThreads, smem>>>(core0, prev0, core, prev, d, reps);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(cycles_host, d, sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}

#include "../qr_std.cuh"
__global__ void __launch_bounds__(kThreads, 1) k_orthblk_probe(const double *core0, const double *prev0, double *core,
                                                               double *prev, long long *out, int reps) {
  extern __shared__ double sm[];
  long long tot = 0;
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < 64 * 128; i += kThreads) { core[i] = core0[i]; prev[i] = prev0[i]; }
    __syncthreads();
    const long long t0 = clock64();
    orth_site_blk(core, 128, 64, prev, 128, sm);
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) out[0] = tot / reps;
}

extern "C" int qtt_probe_blktrace(long long *host) {
  return (int)cudaMemcpyFromSymbol(host, g_blktrace, sizeof(long long) * 8 * 16);
}

extern "C" int qtt_probe_orthblk(const double *core0, const double *prev0, double *core, double *prev,
                                 long long *cycles_host, int reps) {
  long long *d;
  cudaMalloc(&d, sizeof(long long));
  const size_t smem = (size_t)orth_blk_smem() * sizeof(double);
  cudaFuncSetAttribute(k_orthblk_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_orthblk_probe<<<1, kThreads, smem>>>(core0, prev0, core, prev, d, reps);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(cycles_host, d, sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}
