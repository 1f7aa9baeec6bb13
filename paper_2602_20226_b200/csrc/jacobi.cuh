// jacobi.cuh -- a4: one-sided (Hestenes) Jacobi SVD of a site matrix held in shared memory,
// register-blocked for sm_100a ("dotted lines stand for a
// singular value decomposition").
//
// A is m x p (m <= 32*RPL rows, p <= 16*WB columns), column-major in shared memory with
// leading dimension kLdA; rows >= m and columns >= p must be zero.  The 16 column blocks of
// WB columns are paired by a cyclic round-robin over the 8 warps (15 block rounds per
// sweep).  A warp holds its two blocks in registers (lane l owns rows l, l+32, ...), and
// processes WB disjoint column pairs per inner round: 3*WB partial dot products per lane,
// one butterfly reduce-scatter across the warp, rotation parameters computed in parallel
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

template <int RPL, int WB, int MODE, int S>
__device__ __forceinline__ void jac_round(double (&X)[2 * WB][RPL], double tol, int &rot) {
  constexpr int NP = (MODE == 0) ? WB : 2 * (WB / 2);   // pairs in this round
  constexpr int NV = (3 * NP <= 4) ? 4 : (3 * NP <= 8) ? 8 : (3 * NP <= 16) ? 16 : 32;
  const int lane = threadIdx.x & 31;
  double v[NV];
#pragma unroll
  for (int a = 0; a < NP; ++a) {
    const int i = pair_i<WB, MODE, S>(a), j = pair_j<WB, MODE, S>(a);
    double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      al = fma(X[i][t], X[i][t], al);
      be = fma(X[j][t], X[j][t], be);
      ga = fma(X[i][t], X[j][t], ga);
    }
    v[3 * a] = al; v[3 * a + 1] = be; v[3 * a + 2] = ga;
  }
#pragma unroll
  for (int k = 3 * NP; k < NV; ++k) v[k] = 0.0;
  halve<NV, 16, NV>(v, lane);
  const double tot = v[0];
  constexpr int sh = 5 - ilog2<NV>();
  const int a = lane % NP;
  const double al = __shfl_sync(0xffffffffu, tot, (3 * a) << sh);
  const double be = __shfl_sync(0xffffffffu, tot, (3 * a + 1) << sh);
  const double ga = __shfl_sync(0xffffffffu, tot, (3 * a + 2) << sh);
  double c = 1.0, s = 0.0;
  const bool doit = (ga != 0.0) && (fabs(ga) > tol * sqrt(al) * sqrt(be));
  if (doit) {
    const double zeta = (be - al) / (2.0 * ga);
    const double t = (fabs(zeta) > 1e150) ? 0.5 / zeta
                                          : copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
    c = 1.0 / sqrt(fma(t, t, 1.0));
    s = c * t;
  }
  if (__any_sync(0xffffffffu, doit)) rot = 1;
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
}

template <int RPL, int WB, int MODE, int S, int SEND>
__device__ __forceinline__ void jac_rounds(double (&X)[2 * WB][RPL], double tol, int &rot) {
  if constexpr (S < SEND) {
    jac_round<RPL, WB, MODE, S>(X, tol, rot);
    jac_rounds<RPL, WB, MODE, S + 1, SEND>(X, tol, rot);
  }
}

// Returns the number of sweeps executed (== kJacobiMaxSweeps: not converged).
template <int RPL, int WB>
__device__ int jacobi_blocked(double *A, int m, int *flag) {
  constexpr int NB = 2 * kWarps;      // 16 blocks of WB columns
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double tol = (double)max(m, 1) * DBL_EPSILON;
  double X[2 * WB][RPL];
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
      if constexpr (WB > 1) {
        if (r == 0) jac_rounds<RPL, WB, 1, 0, WB - 1>(X, tol, rot);
      }
      jac_rounds<RPL, WB, 0, 0, WB>(X, tol, rot);
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
__device__ __forceinline__ int jacobi_dispatch(double *A, int m, int p, int *flag) {
  const int rpl = (m <= 32) ? 1 : (m <= 64) ? 2 : 4;
  const int wb = (p <= 16) ? 1 : (p <= 32) ? 2 : (p <= 64) ? 4 : 8;
#define QTT_JAC(R, W) if (rpl == R && wb == W) return jacobi_blocked<R, W>(A, m, flag);
  QTT_JAC(1, 1) QTT_JAC(1, 2) QTT_JAC(1, 4) QTT_JAC(1, 8)
  QTT_JAC(2, 1) QTT_JAC(2, 2) QTT_JAC(2, 4) QTT_JAC(2, 8)
  QTT_JAC(4, 1) QTT_JAC(4, 2) QTT_JAC(4, 4) QTT_JAC(4, 8)
#undef QTT_JAC
  return kJacobiMaxSweeps;
}

}  // namespace qtt
