// jacobi.cuh -- a4: one-sided (Hestenes) Jacobi SVD of a site matrix held in shared memory,
// register-blocked for sm_100a ("dotted lines stand for a
// singular value decomposition").
//
// A is m x p (m <= 32*RPL rows, p <= 16*WB columns), column-major in shared memory with
// leading dimension kLdA; rows >= m and columns >= p must be zero.  The 16 column blocks of
// WB columns are paired by a cyclic round-robin over the 8 warps (15 block rounds per
// sweep).  A warp holds its two blocks in registers (lane l owns rows l, l+32, ...), and
// processes WB disjoint column pairs per inner round: WB partial dot products per lane,
// one butterfly reduce-scatter across the warp (column norms are tracked in shared memory
// by the rotation identities), rotation parameters computed in parallel
// (one pair per lane), broadcast by shuffles, rotations applied in registers.  Every pair of
// columns is visited exactly once per sweep (cross pairs for every block pair, intra-block
// pairs in the first block round).  Converged when no pair needed a rotation, i.e.
// |a_i.a_j| <= m*eps*|a_i||a_j| for all i < j.
#pragma once
#include "common.cuh"

namespace qtt {

constexpr int kJacobiMaxSweeps = 60;

// Butterfly reduce-scatter: NV (power of two <= 32) per-lane partial sums -> lane l holds the
// warp total of value index (l >> (5 - log2 NV)) in v[0].
template <int CNT, int OFF, int NV>
__device__ __forceinline__ void halve(double (&v)[NV], int lane) {
  if constexpr (CNT > 1) {
    const bool up = (lane & OFF) != 0;
#pragma unroll
    for (int k = 0; k < CNT / 2; ++k) {
      const double send = up ? v[k] : v[k + CNT / 2];
      const double keep = up ? v[k + CNT / 2] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
    }
    halve<CNT / 2, OFF / 2, NV>(v, lane);
  } else {
    double r = v[0];
#pragma unroll
    for (int o = OFF; o >= 1; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    v[0] = r;
  }
}

template <int N>
__device__ constexpr int ilog2() { return N <= 1 ? 0 : 1 + ilog2<N / 2>(); }

// Pair a of an inner round.  MODE 0: cross pairs (a, WB + (a+S)%WB).  MODE 1: intra-block
// pairs of round S of the circle method on WB players, in block I for a < WB/2, else in J.
template <int WB, int MODE, int S>
__device__ constexpr int pair_i(int a) {
  if (MODE == 0) return a;
  const int h = WB / 2, t = (a < h) ? a : a - h, base = (a < h) ? 0 : WB;
  const int k = t;
  return base + ((k == 0) ? 0 : 1 + (k - 1 + S) % (WB > 1 ? WB - 1 : 1));
}
template <int WB, int MODE, int S>
__device__ constexpr int pair_j(int a) {
  if (MODE == 0) return WB + (a + S) % WB;
  const int h = WB / 2, t = (a < h) ? a : a - h, base = (a < h) ? 0 : WB;
  const int k = WB - 1 - t;
  return base + ((k == 0) ? 0 : 1 + (k - 1 + S) % (WB > 1 ? WB - 1 : 1));
}

// Exact squared norms of the warp's 2*WB register columns -> nrm[0..2WB) (shared, per warp).
template <int RPL, int WB>
__device__ __forceinline__ void warp_norms(const double (&X)[2 * WB][RPL], double *nrm) {
  constexpr int NC = 2 * WB;
  constexpr int NV = (NC <= 4) ? 4 : (NC <= 8) ? 8 : (NC <= 16) ? 16 : 32;
  const int lane = threadIdx.x & 31;
  double v[NV];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < RPL; ++t) s = fma(X[c][t], X[c][t], s);
    v[c] = s;
  }
#pragma unroll
  for (int k = NC; k < NV; ++k) v[k] = 0.0;
  halve<NV, 16, NV>(v, lane);
  constexpr int sh = 5 - ilog2<NV>();
  if ((lane & ((1 << sh) - 1)) == 0 && (lane >> sh) < NC) nrm[lane >> sh] = v[0];
  __syncwarp();
}

// One inner round: NP disjoint column pairs.  Column norms come from nrm[] (kept up to date
// by the exact rotation identities a' = a - t*g, b' = b + t*g, refreshed exactly when a
// norm collapses by more than sqrt(eps), as in LAPACK dgesvj); only the NP cross dot
// products g are reduced across the warp.
template <int RPL, int WB, int MODE, int S>
__device__ __forceinline__ void jac_round(double (&X)[2 * WB][RPL], double *nrm, double tol, int &rot) {
  constexpr int NP = (MODE == 0) ? WB : 2 * (WB / 2);   // pairs in this round
  constexpr int NV = (NP <= 4) ? 4 : (NP <= 8) ? 8 : (NP <= 16) ? 16 : 32;
  const int lane = threadIdx.x & 31;
  double v[NV];
#pragma unroll
  for (int a = 0; a < NP; ++a) {
    const int i = pair_i<WB, MODE, S>(a), j = pair_j<WB, MODE, S>(a);
    double g0 = 0.0, g1 = 0.0;
#pragma unroll
    for (int t = 0; t < RPL; t += 2) {
      g0 = fma(X[i][t], X[j][t], g0);
      if (t + 1 < RPL) g1 = fma(X[i][t + 1], X[j][t + 1], g1);
    }
    v[a] = g0 + g1;
  }
#pragma unroll
  for (int k = NP; k < NV; ++k) v[k] = 0.0;
  halve<NV, 16, NV>(v, lane);
  constexpr int sh = 5 - ilog2<NV>();
  const int a = lane % NP;
  const double ga = __shfl_sync(0xffffffffu, v[0], a << sh);
  int ia = 0, ja = 0;
#pragma unroll
  for (int k = 0; k < NP; ++k)
    if (a == k) { ia = pair_i<WB, MODE, S>(k); ja = pair_j<WB, MODE, S>(k); }
  const double al = nrm[ia], be = nrm[ja];
  // Rotation angle (Rutishauser): t = sign(d) 2g / (|d| + sqrt(d^2 + 4g^2)), d = b - a;
  // c = 1/sqrt(1+t^2), s = c t.  Rotate only if |g| > tol sqrt(a b) (squared test).
  const double d = be - al;
  const double g2 = ga + ga;
  const bool doit = (ga * ga > (tol * tol) * (al * be)) && (al > 0.0) && (be > 0.0);
  const double h = sqrt(fma(d, d, g2 * g2));
  const double den = fabs(d) + h;
  const double t = doit ? copysign(1.0, d) * g2 * __drcp_rn(den) : 0.0;
  const double c = rsqrt(fma(t, t, 1.0));
  const double s = c * t;
  const double al2 = doit ? fma(-t, ga, al) : al;
  const double be2 = doit ? fma(t, ga, be) : be;
  const bool collapse = doit && (al2 < 1.5e-8 * al || be2 < 1.5e-8 * be);
  if (__any_sync(0xffffffffu, doit)) rot = 1;
  __syncwarp();
  if (lane < NP) { nrm[ia] = al2; nrm[ja] = be2; }
#pragma unroll
  for (int a2 = 0; a2 < NP; ++a2) {
    const int i = pair_i<WB, MODE, S>(a2), j = pair_j<WB, MODE, S>(a2);
    const double ca = __shfl_sync(0xffffffffu, c, a2), sa = __shfl_sync(0xffffffffu, s, a2);
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const double x = X[i][t], y = X[j][t];
      X[i][t] = fma(ca, x, -sa * y);
      X[j][t] = fma(sa, x, ca * y);
    }
  }
  __syncwarp();
  if (__any_sync(0xffffffffu, collapse)) warp_norms<RPL, WB>(X, nrm);   // cancellation: refresh exactly
}

template <int RPL, int WB, int MODE, int S, int SEND>
__device__ __forceinline__ void jac_rounds(double (&X)[2 * WB][RPL], double *nrm, double tol, int &rot) {
  if constexpr (S < SEND) {
    jac_round<RPL, WB, MODE, S>(X, nrm, tol, rot);
    jac_rounds<RPL, WB, MODE, S + 1, SEND>(X, nrm, tol, rot);
  }
}

// Returns the number of sweeps executed (== kJacobiMaxSweeps: not converged).
template <int RPL, int WB>
__device__ int jacobi_blocked(double *A, int m, int *flag, double *nrm_all) {
  constexpr int NB = 2 * kWarps;      // 16 blocks of WB columns
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double tol = (double)max(m, 1) * DBL_EPSILON;
  double X[2 * WB][RPL];
  double *nrm = nrm_all + warp * 2 * WB;
  int sweep = 0;
  for (; sweep < kJacobiMaxSweeps; ++sweep) {
    int rot = 0;
    for (int r = 0; r < NB - 1; ++r) {
      const int kI = warp, kJ = NB - 1 - warp;                      // circle method positions
      const int I = (kI == 0) ? 0 : 1 + (kI - 1 + r) % (NB - 1);
      const int J = 1 + (kJ - 1 + r) % (NB - 1);
#pragma unroll
      for (int c = 0; c < WB; ++c)
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          X[c][t] = A[(size_t)(I * WB + c) * kLdA + lane + 32 * t];
          X[WB + c][t] = A[(size_t)(J * WB + c) * kLdA + lane + 32 * t];
        }
      warp_norms<RPL, WB>(X, nrm);
      if constexpr (WB > 1) {
        if (r == 0) jac_rounds<RPL, WB, 1, 0, WB - 1>(X, nrm, tol, rot);
      }
      jac_rounds<RPL, WB, 0, 0, WB>(X, nrm, tol, rot);
#pragma unroll
      for (int c = 0; c < WB; ++c)
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          A[(size_t)(I * WB + c) * kLdA + lane + 32 * t] = X[c][t];
          A[(size_t)(J * WB + c) * kLdA + lane + 32 * t] = X[WB + c][t];
        }
      __syncthreads();
    }
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    if (lane == 0 && rot) *flag = 1;
    __syncthreads();
    const int any = *flag;
    __syncthreads();
    if (!any) { ++sweep; break; }
  }
  return sweep;
}

// Dispatch on the padded sizes: RPL = ceil(m/32) in {1,2,4}, WB = ceil(p/16) in {1,2,4,8}.
__device__ __forceinline__ int jacobi_dispatch(double *A, int m, int p, int *flag, double *nrm_all) {
  const int rpl = (m <= 32) ? 1 : (m <= 64) ? 2 : 4;
  const int wb = (p <= 16) ? 1 : (p <= 32) ? 2 : (p <= 64) ? 4 : 8;
#define QTT_JAC(R, W) if (rpl == R && wb == W) return jacobi_blocked<R, W>(A, m, flag, nrm_all);
  QTT_JAC(1, 1) QTT_JAC(1, 2) QTT_JAC(1, 4) QTT_JAC(1, 8)
  QTT_JAC(2, 1) QTT_JAC(2, 2) QTT_JAC(2, 4) QTT_JAC(2, 8)
  QTT_JAC(4, 1) QTT_JAC(4, 2) QTT_JAC(4, 4) QTT_JAC(4, 8)
#undef QTT_JAC
  return kJacobiMaxSweeps;
}

}  // namespace qtt
