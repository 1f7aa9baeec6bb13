// common.cuh -- shared helpers for libqtt (sm_100a, float64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <cfloat>

#include "../../include/qtt.h"

namespace qtt {

constexpr int kThreads = 256;     // CTA size of every per-member kernel (8 warps)
constexpr int kWarps = kThreads / 32;
// c-A31: Jacobi may leave columns of squared norm <= eps_mach^2 ||A||_F^2 unrotated
// only when the truncation discards them for certain: their total mass p eps_mach^2 ||A||_F^2
// must stay below the rule's budget eps^2 ||A||_F^2, i.e. eps^2 > p eps_mach^2 (and eps > 1e-14,
// the threshold the rule was measured with).  p: the matrix's column count (or an upper bound).
__host__ __device__ __forceinline__ bool noise_ok(double eps, int p) {
  return eps > 1e-14 && eps * eps > (double)p * (DBL_EPSILON * DBL_EPSILON);
}
constexpr int kLdA = 129;         // leading dim of the shared R / Jacobi matrix (odd: no bank conflicts)

void set_error(const char *fmt, ...);
qtt_status_t cuda_status(cudaError_t e, const char *what);

#define QTT_CUDA_TRY(expr)                                           \
  do {                                                               \
    cudaError_t _e = (expr);                                         \
    if (_e != cudaSuccess) return ::qtt::cuda_status(_e, #expr);     \
  } while (0)

// ------------------------------------------------------------------ device helpers

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum over NW warps; `red` is >= NW doubles of shared memory.
// All threads must call it; returns the total to every thread.
template <int NW = kWarps>
__device__ __forceinline__ double block_sum(double v, double *red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) t += red[w];   // fixed order: deterministic
  return t;
}

// CTA-wide C = A * B (+ C if accumulate) with element accessors.  64x64 output tiles,
// 16-deep K chunks staged in shared memory `sm` (>= 2*16*64 doubles); 256 threads,
// each owning a 4x4 register tile (rows ty+16i, cols tx+16j: conflict-free smem reads).
// A(m,k), B(k,n) are callables returning double; store(m,n,v) writes the result.
// NT threads (256: 64x64 tiles; 512: 64x128 tiles), staging >= 16*64 + 16*TN doubles.
template <int NT = kThreads, typename FA, typename FB, typename FS>
__device__ void cta_gemm(int M, int N, int K, FA A, FB B, FS store, double *sm) {
  static_assert(NT == 256 || NT == 512, "cta_gemm: 256 or 512 threads");
  constexpr int TN = (NT == 512) ? 128 : 64, TX = TN / 4;
  double *As = sm;            // [16][64]
  double *Bs = sm + 16 * 64;  // [16][TN]
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  for (int m0 = 0; m0 < M; m0 += 64) {
    for (int n0 = 0; n0 < N; n0 += TN) {
      double acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
      for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
        for (int e = 0; e < 1024 / NT; ++e) {
          const int idx = tid + e * NT;            // 0..1023
          const int kk = idx >> 6, mm = idx & 63;
          const int gm = m0 + mm, gk = k0 + kk;
          As[kk * 64 + mm] = (gm < M && gk < K) ? A(gm, gk) : 0.0;
        }
#pragma unroll
        for (int e = 0; e < 16 * TN / NT; ++e) {
          const int idx = tid + e * NT;            // 0..16*TN-1
          const int kk = idx / TN, nn = idx % TN;
          const int gn = n0 + nn, gk = k0 + kk;
          Bs[kk * TN + nn] = (gn < N && gk < K) ? B(gk, gn) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          double a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) a[i] = As[kk * 64 + ty + 16 * i];
#pragma unroll
          for (int j = 0; j < 4; ++j) b[j] = Bs[kk * TN + tx + TX * j];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int gm = m0 + ty + 16 * i, gn = n0 + tx + TX * j;
          if (gm < M && gn < N) store(gm, gn, acc[i][j]);
        }
    }
  }
}

// Branch-free reciprocal and reciprocal square root: MUFU seed + 2 Newton steps.  The seed's
// relative error is <= 1e-6 (measured over 2^-40..2^40 by csrc/probe/lat.cu), so two
// quadratic steps give ~1e-24 << 2^-53: full fp64 accuracy for the normal range used here.
// (Rotation parameters need c^2+s^2 = 1 to working precision, which s = c*t with
// c = rsqrt(1+t^2) guarantees.)
#ifndef QTT_RSQRT_HALLEY
#define QTT_RSQRT_HALLEY 1
#endif

__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#if QTT_RSQRT_HALLEY
  // one third-order step y (1 + e + e^2), e = 1 - x y: error ~e^3 ~ 1e-18 << 2^-53
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
#else
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
#endif
}
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#if QTT_RSQRT_HALLEY
  // one third-order step: y (1 + e/2 + 3e^2/8), e = 1 - x y^2; seed error <= 1e-6 leaves
  // ~(5/16) e^3 ~ 3e-19 << 2^-53 -- one dependent step shorter than two Newton steps
  const double h = x * y;
  const double e = fma(-h, y, 1.0);
  const double t = fma(0.375, e, 0.5);
  const double ye = y * e;
  return fma(ye, t, y);
#else
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const double h = x * y;
    const double e = fma(-h, y, 1.0);      // 1 - x y^2
    y = fma(0.5 * y, e, y);
  }
  return y;
#endif
}

// LAPACK dlarfg convention: x = [alpha; x2], ||x2||^2 = xnorm2.  Returns tau and beta and
// the scale 1/(alpha - beta) for v2 = x2 * scale (v0 = 1 implicit).  H x = [beta; 0].
__device__ __forceinline__ void householder(double alpha, double xnorm2, double &tau, double &beta,
                                            double &scale) {
  if (xnorm2 == 0.0) {
    tau = 0.0; beta = alpha; scale = 0.0;
    return;
  }
  const double nrm = sqrt(alpha * alpha + xnorm2);
  beta = (alpha >= 0.0) ? -nrm : nrm;
  tau = (beta - alpha) / beta;
  scale = 1.0 / (alpha - beta);
}

// the rare path of householder_fast<true> out of line (IEEE sqrt and divisions inlined into
// every unrolled panel column only cost instruction-cache space)
static __device__ __noinline__ void householder_slow(double alpha, double xnorm2, double &tau, double &beta, double &scale) {
  householder(alpha, xnorm2, tau, beta, scale);
}

// householder() with MUFU-seeded Newton rcp / rsqrt instead of IEEE sqrt and two divisions
// (same values to a few ulps; shortens the serial chain of a panel factorisation).
// tau = (beta - alpha)/beta = 1 + |alpha|/nrm;  scale = 1/(alpha - beta) = sign(alpha)/(|alpha| + nrm).
template <bool OOL = false>
__device__ __forceinline__ void householder_fast(double alpha, double xnorm2, double &tau, double &beta,
                                                 double &scale) {
  const double a2 = fma(alpha, alpha, xnorm2);
  if (xnorm2 == 0.0 || !(a2 > 1e-280 && a2 < 1e280)) {   // zero column / outside the ftz-safe range
    if (OOL) householder_slow(alpha, xnorm2, tau, beta, scale);
    else householder(alpha, xnorm2, tau, beta, scale);
    return;
  }
  const double rn = fast_rsqrt(a2);
  const double nrm = a2 * rn;
  const double aa = fabs(alpha);
  beta = (alpha >= 0.0) ? -nrm : nrm;
  tau = fma(aa, rn, 1.0);
  const double sc = fast_rcp(aa + nrm);
  scale = (alpha >= 0.0) ? sc : -sc;
}


// ---- TMA bulk copies (cp.async.bulk, the async proxy) with an mbarrier transaction count ----
__device__ __forceinline__ uint32_t tma_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tma_mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tma_smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// generic-proxy shared-memory accesses before this point are ordered before later async-proxy
// (TMA) accesses of the CTA
__device__ __forceinline__ void tma_fence_proxy() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tma_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tma_smem_u32(bar)), "r"(bytes) : "memory");
}
// global -> shared, bytes a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(tma_smem_u32(dst)), "l"(src), "r"(bytes), "r"(tma_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "TMAW_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra TMAW_%=;\n\t}" ::"r"(tma_smem_u32(bar)), "r"(parity) : "memory");
}

}  // namespace qtt
