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
#ifndef QTT_JAC_PROFILE
#define QTT_JAC_PROFILE 0
#endif
#if QTT_JAC_PROFILE
// diagnostics build only: cycles per jac_round phase summed over warp 0 of every CTA
// [0] dots + reduce-scatter, [1] rotation parameters, [2] rotation, [3] rounds
__device__ unsigned long long g_jprof[24];   // [4..11]: qr_of_TH phases (qr_small.cuh), [12..15] a1, [16..19] a2
#define QTT_JPROF_T(v) const long long v = clock64()
#define QTT_JPROF_ADD(i, d) if (threadIdx.x == 0) atomicAdd(&g_jprof[i], (unsigned long long)(d))
#else
#define QTT_JPROF_T(v)
#define QTT_JPROF_ADD(i, d)
#endif
#ifndef QTT_JAC_SCALED
// scaled (fast-Givens, Anda-Park) rotations: two DFMA per row and pair instead of two DMUL + two
// DFMA; the rotation phase of a round runs both warps of an SMSP on the FP64 pipe at once, so
// halving its FP64 instructions shortens the round (round 2: 131.2k -> 133.4k site-steps/s on
// cfg5; round 1, before the division-free angles and the Halley rsqrt, measured no change)
#define QTT_JAC_SCALED 1
#endif
#ifndef QTT_JAC_GRAMCHECK
#define QTT_JAC_GRAMCHECK 1
#endif
#ifndef QTT_JAC_DIVFREE
#define QTT_JAC_DIVFREE 1
#endif
#ifndef QTT_JAC_SMEMBC
#define QTT_JAC_SMEMBC 1
#endif
#ifndef QTT_JAC_UNROLL
#define QTT_JAC_UNROLL 4
#endif

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
__host__ __device__ constexpr int ilog2() { return N <= 1 ? 0 : 1 + ilog2<N / 2>(); }

// Exact squared norms of the warp's 2*WB register columns -> nrm[0..2WB) (shared, per warp).
template <int RPL, int WB>
__device__ __forceinline__ void warp_norms(const double (&X)[2 * WB][RPL], double *nrm, const double *dsc,
                                           const int *slot_col) {
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
  if ((lane & ((1 << sh) - 1)) == 0 && (lane >> sh) < NC) {
    const int col = slot_col[lane >> sh];
#if QTT_JAC_SCALED
    nrm[col] = v[0] * (dsc[col] * dsc[col]);
#else
    nrm[col] = v[0];
#endif
  }
  __syncwarp();
}

// One inner round on NP fixed register pairs (P0 + a, P1 + a*D1 ... see pair_slots):
//   MODE 0 (cross):  pairs (a, WB + a),              a < WB
//   MODE 1 (intra):  pairs (t, WB-1-t), (WB+t, 2WB-1-t), t < WB/2
// The caller rotates registers between rounds so that these fixed slots walk through the
// round-robin orderings.  slot_col[k] maps register slot k to its column's norm index.
template <int WB, int MODE, int SH = 0>
__device__ __forceinline__ constexpr int slot_i(int a) {
  return MODE != 1 ? a : (a < WB / 2 ? a : WB + (a - WB / 2));
}
template <int WB, int MODE, int SH = 0>
__device__ __forceinline__ constexpr int slot_j(int a) {
  return MODE == 0 ? WB + (a + SH) % WB                 // cross round SH J positions further
                   : (a < WB / 2 ? WB - 1 - a : 2 * WB - 1 - (a - WB / 2));
}

template <int RPL, int WB, int MODE, int SH = 0>
__device__ __forceinline__ void jac_round(double (&X)[2 * WB][RPL], double *nrm, double *dsc, double *esc,
                                          double2 *csb, const int *slot_col, double tol, double noise, int &rot) {
  constexpr int NP = (MODE != 1) ? WB : 2 * (WB / 2);   // pairs in this round
  constexpr int NV = (NP <= 4) ? 4 : (NP <= 8) ? 8 : (NP <= 16) ? 16 : 32;
  const int lane = threadIdx.x & 31;
  QTT_JPROF_T(jt0);
  double v[NV];
#pragma unroll
  for (int a = 0; a < NP; ++a) {
    const int i = slot_i<WB, MODE, SH>(a), j = slot_j<WB, MODE, SH>(a);
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
  int si = 0, sj = 0;
#pragma unroll
  for (int k = 0; k < NP; ++k)
    if (a == k) { si = slot_i<WB, MODE, SH>(k); sj = slot_j<WB, MODE, SH>(k); }
  const int ci = slot_col[si], cj = slot_col[sj];
  const double al = nrm[ci], be = nrm[cj];
#if QTT_JAC_SCALED
  const double di = dsc[ci], dj = dsc[cj], ei = esc[ci], ej = esc[cj];
  const double ga = __shfl_sync(0xffffffffu, v[0], a << sh) * (di * dj);   // true a_i . a_j
#else
  const double ga = __shfl_sync(0xffffffffu, v[0], a << sh);
#endif
  QTT_JPROF_T(jt1);
  // Rotation angle (Rutishauser): t = sign(d) 2g / (|d| + sqrt(d^2 + 4g^2)), d = b - a;
  // c = 1/sqrt(1+t^2), s = c t.  Rotate only if |g| > tol sqrt(a b) (squared test).
  const double d = be - al;
  const double g2 = ga + ga;
  // noise = eps^2 ||A||_F^2: a column at rounding-noise level is treated as converged (its
  // relative orthogonality is below fp64 resolution; see large.cu rot_pair)
  const double x2 = fma(d, d, g2 * g2);
  // x2 >= DBL_MIN: the MUFU rsqrt seed flushes a subnormal argument to zero.  jacobi_blocked
  // scales A so ||A||_F^2 is in [1, 4), so only columns below ~1e-150 relative can fail this
  const bool doit = (ga * ga > (tol * tol) * (al * be)) && (al > noise) && (be > noise) && (x2 >= DBL_MIN);
#if QTT_JAC_DIVFREE
  // same angle without a division: y = 1/sqrt(d^2 + 4 g^2), c^2 = (1 + |d| y)/2, z = 1/c,
  // s = sign(d) g y z, t = s z
  // the angle depends on d : g only; below ~1e-280 the MUFU seed of rsqrt would flush the
  // (subnormal) argument to zero, so tiny pairs (exact sweeps, noise = 0) are rescaled first
  const double y = doit ? fast_rsqrt(x2) : 0.0;
  const double c2 = doit ? fma(0.5 * fabs(d), y, 0.5) : 1.0;
  const double z = doit ? fast_rsqrt(c2) : 1.0;
  const double c = c2 * z;
  const double s = copysign(1.0, d) * ga * y * z;
  const double t = s * z;
#else
  const double h = doit ? x2 * fast_rsqrt(x2) : 1.0;
  const double den = fabs(d) + h;
  const double t = doit ? copysign(1.0, d) * g2 * fast_rcp(den) : 0.0;
  const double c = fast_rsqrt(fma(t, t, 1.0));
  const double s = c * t;
#endif
  const double al2 = doit ? fma(-t, ga, al) : al;
  const double be2 = doit ? fma(t, ga, be) : be;
  const bool collapse = doit && (al2 < 1.5e-8 * al || be2 < 1.5e-8 * be);
  if (__any_sync(0xffffffffu, doit)) rot |= 1;
#if QTT_JAC_GRAMCHECK
  // bit 1: some pair of this sweep was still far from converged (|cos| >= 1e-6), so the
  // next sweep cannot be skipped by the Gram check (jacobi_blocked)
  if (__any_sync(0xffffffffu, al > noise && be > noise && ga * ga >= 1e-12 * (al * be))) rot |= 2;
#endif
  __syncwarp();
  QTT_JPROF_T(jt2);
#if QTT_JAC_SCALED
  // scaled (Anda-Park) rotation: true column = dsc * register column; the register columns
  // take X_i -= t (d_j/d_i) X_j, X_j += t (d_i/d_j) X_i and the scales take the cosine
#if !QTT_JAC_DIVFREE
  const double z = fma(t, t, 1.0) * c;                 // 1/c
#endif
  const double t1 = t * (dj * ei), t2 = t * (di * ej);
  if (lane < NP) {
    nrm[ci] = al2; nrm[cj] = be2;
    dsc[ci] = di * c; dsc[cj] = dj * c; esc[ci] = ei * z; esc[cj] = ej * z;
    csb[lane] = make_double2(t1, t2);
  }
  (void)s;
  __syncwarp();
#pragma unroll
  for (int a2 = 0; a2 < NP; ++a2) {
    const int i = slot_i<WB, MODE, SH>(a2), j = slot_j<WB, MODE, SH>(a2);
    const double2 tt2 = csb[a2];
    const double u1 = tt2.x, u2 = tt2.y;
#pragma unroll
    for (int tt = 0; tt < RPL; ++tt) {
      const double x = X[i][tt], y = X[j][tt];
      X[i][tt] = fma(-u1, y, x);
      X[j][tt] = fma(u2, x, y);
    }
  }
#elif QTT_JAC_SMEMBC
  // (c, s) of every pair through shared memory: one 16-byte store per pair, one broadcast
  // 16-byte load per pair and lane (instead of two 64-bit shuffles per pair)
  if (lane < NP) { nrm[ci] = al2; nrm[cj] = be2; csb[lane] = make_double2(c, s); }
  __syncwarp();
#pragma unroll
  for (int a2 = 0; a2 < NP; ++a2) {
    const int i = slot_i<WB, MODE, SH>(a2), j = slot_j<WB, MODE, SH>(a2);
    const double2 cs2 = csb[a2];
    const double ca = cs2.x, sa = cs2.y;
#pragma unroll
    for (int tt = 0; tt < RPL; ++tt) {
      const double x = X[i][tt], y = X[j][tt];
      X[i][tt] = fma(ca, x, -sa * y);
      X[j][tt] = fma(sa, x, ca * y);
    }
  }
#else
  if (lane < NP) { nrm[ci] = al2; nrm[cj] = be2; }
#pragma unroll
  for (int a2 = 0; a2 < NP; ++a2) {
    const int i = slot_i<WB, MODE, SH>(a2), j = slot_j<WB, MODE, SH>(a2);
    const double ca = __shfl_sync(0xffffffffu, c, a2), sa = __shfl_sync(0xffffffffu, s, a2);
#pragma unroll
    for (int tt = 0; tt < RPL; ++tt) {
      const double x = X[i][tt], y = X[j][tt];
      X[i][tt] = fma(ca, x, -sa * y);
      X[j][tt] = fma(sa, x, ca * y);
    }
  }
#endif
  __syncwarp();
  QTT_JPROF_T(jt3);
  QTT_JPROF_ADD(0, jt1 - jt0); QTT_JPROF_ADD(1, jt2 - jt1); QTT_JPROF_ADD(2, jt3 - jt2); QTT_JPROF_ADD(3, 1);
  if (__any_sync(0xffffffffu, collapse)) warp_norms<RPL, WB>(X, nrm, dsc, slot_col);   // refresh exactly
}

// Shift the J block by S positions at once (after S fixed-slot cross rounds with shifts
// 0..S-1): each register moves once per S rounds.
template <int RPL, int WB, int S>
__device__ __forceinline__ void rotate_Jn(double (&X)[2 * WB][RPL], int *slot_col) {
#pragma unroll
  for (int t = 0; t < RPL; ++t) {
    double f[S];
#pragma unroll
    for (int e = 0; e < S; ++e) f[e] = X[WB + e][t];
#pragma unroll
    for (int a = 0; a < WB - S; ++a) X[WB + a][t] = X[WB + a + S][t];
#pragma unroll
    for (int e = 0; e < S; ++e) X[2 * WB - S + e][t] = f[e];
  }
  if ((threadIdx.x & 31) == 0) {
    int f[S];
    for (int e = 0; e < S; ++e) f[e] = slot_col[WB + e];
    for (int a = 0; a < WB - S; ++a) slot_col[WB + a] = slot_col[WB + a + S];
    for (int e = 0; e < S; ++e) slot_col[2 * WB - S + e] = f[e];
  }
  __syncwarp();
}

template <int RPL, int WB, int SH, int U>
__device__ __forceinline__ void cross_rounds(double (&X)[2 * WB][RPL], double *nrm, double *dsc, double *esc,
                                             double2 *csb, const int *slot_col, double tol, double noise, int &rot) {
  if constexpr (SH < U) {
    jac_round<RPL, WB, 0, SH>(X, nrm, dsc, esc, csb, slot_col, tol, noise, rot);
    cross_rounds<RPL, WB, SH + 1, U>(X, nrm, dsc, esc, csb, slot_col, tol, noise, rot);
  }
}

template <int RPL, int WB>
__device__ __forceinline__ void rotate_circle(double (&X)[2 * WB][RPL], int *slot_col) {
  // circle method inside each block: position 0 fixed, positions 1..WB-1 rotate by one
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int o = h * WB;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const double first = X[o + 1][t];
#pragma unroll
      for (int k = 1; k < WB - 1; ++k) X[o + k][t] = X[o + k + 1][t];
      X[o + WB - 1][t] = first;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    for (int h = 0; h < 2; ++h) {
      const int o = h * WB;
      const int f = slot_col[o + 1];
      for (int k = 1; k < WB - 1; ++k) slot_col[o + k] = slot_col[o + k + 1];
      slot_col[o + WB - 1] = f;
    }
  }
  __syncwarp();
}

// True iff |a_i . a_j| <= tolg * |a_i| |a_j| for every pair of the first pc columns of A (column-
// major, leading dimension kLdA, 32*RPL rows, zero padding beyond the matrix).  Column norms by
// warp reductions, off-diagonal Gram entries by DMMA (m8n8k4) over the upper-triangular 8 x 8
// tiles.  All threads call it; uses scratch[0 .. 128) and *flag.
__device__ __forceinline__ void dmma884_j(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int NW, int RPL>
__device__ bool gram_converged(const double *A, int pc, double tolg, double noise, double *scratch, int *flag) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *nn = scratch;                         // [128] squared column norms
  for (int j = warp; j < pc; j += NW) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < RPL; ++t) { const double v = A[(size_t)j * kLdA + lane + 32 * t]; s = fma(v, v, s); }
    s = warp_sum(s);
    if (lane == 0) nn[j] = s;
  }
  if (threadIdx.x == 0) *flag = 0;
  __syncthreads();
  const int gr = lane >> 2, gc = lane & 3, nt = pc >> 3;
  const double tol2 = tolg * tolg;
  bool bad = false;
  for (int t = warp; t < nt * (nt + 1) / 2; t += NW) {
    int ti = 0, rem = t;                        // t -> (ti <= tj) upper-triangular tile
    while (rem >= nt - ti) { rem -= nt - ti; ++ti; }
    const int tj = ti + rem;
    double c0 = 0.0, c1 = 0.0;
    const double *ai = A + (size_t)(ti * 8 + gr) * kLdA, *aj = A + (size_t)(tj * 8 + gr) * kLdA;
#pragma unroll 8
    for (int k0 = 0; k0 < 32 * RPL; k0 += 4) dmma884_j(c0, c1, ai[k0 + gc], aj[k0 + gc]);
    const int i = ti * 8 + gr;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int j = tj * 8 + 2 * gc + e;
      const double g = e ? c1 : c0;
      if (j > i && nn[i] > noise && nn[j] > noise && g * g > tol2 * (nn[i] * nn[j])) bad = true;
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
  __syncthreads();
  const bool ok = (*flag == 0);
  __syncthreads();
  return ok;
}

// Returns the number of sweeps executed (== kJacobiMaxSweeps: not converged).
// noise_ok: the caller truncates with eps > 1e-14, so columns at rounding-noise level can
// never be kept and need not be orthogonalised (eps = 0 keeps them: they must be orthonormal)
template <int RPL, int WB, int NW>
__device__ int jacobi_blocked(double *A, int m, int *flag, double *scratch, bool noise_ok) {
  constexpr int NB = 2 * NW;          // 2*NW blocks of WB columns (one block pair per warp)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double tol = (double)max(m, 1) * DBL_EPSILON;
  double X[2 * WB][RPL];
  double *nrm = scratch + warp * 2 * WB;                                   // norms by local column
  double *dsc = scratch + NW * 2 * WB + warp * 2 * WB;                     // column scales (scaled rotations)
  double *esc = scratch + NW * 4 * WB + warp * 2 * WB;                     // 1 / column scales
  int *slot_col = reinterpret_cast<int *>(scratch + NW * 6 * WB) + warp * 2 * WB;
  double2 *csb = reinterpret_cast<double2 *>(scratch + NW * 8 * WB + warp * 2 * WB);   // rotation broadcast
  double noise;                                                            // eps^2 ||A||_F^2
  double scale = 1.0;
  {
    double sq = 0.0;
    for (int idx = threadIdx.x; idx < 2 * NW * WB * 32 * RPL; idx += NW * 32) {
      const double v = A[(size_t)(idx / (32 * RPL)) * kLdA + idx % (32 * RPL)];
      sq = fma(v, v, sq);
    }
    sq = warp_sum(sq);
    __syncthreads();
    if (lane == 0) scratch[warp] = sq;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) tot += scratch[w];             // fixed order: deterministic
    // exact power-of-two scaling to ||A||_F^2 in [1, 4) (undone after the sweeps): keeps
    // d^2 + 4 g^2 of every non-negligible pair clear of the subnormal range (jac_round)
    if (tot > 0.0 && isfinite(tot)) {
      const int e = -(ilogb(tot) >> 1);
      if (e != 0) {
        scale = ldexp(1.0, e);
        tot = ldexp(tot, 2 * e);
      }
    }
    noise = noise_ok ? DBL_EPSILON * DBL_EPSILON * tot : 0.0;
    __syncthreads();
    if (scale != 1.0)
      for (int idx = threadIdx.x; idx < 2 * NW * WB * 32 * RPL; idx += NW * 32)
        A[(size_t)(idx / (32 * RPL)) * kLdA + idx % (32 * RPL)] *= scale;
    __syncthreads();
  }
  int sweep = 0;
  for (; sweep < kJacobiMaxSweeps; ++sweep) {
    int rot = 0;
#pragma unroll 1
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
      if (lane < 2 * WB) { slot_col[lane] = lane; dsc[lane] = 1.0; esc[lane] = 1.0; }
      __syncwarp();
      warp_norms<RPL, WB>(X, nrm, dsc, slot_col);
      if constexpr (WB > 1) {
        if (r == 0) {
#pragma unroll 1
          for (int u = 0; u < WB - 1; ++u) {
            jac_round<RPL, WB, 1>(X, nrm, dsc, esc, csb, slot_col, tol, noise, rot);
            rotate_circle<RPL, WB>(X, slot_col);
          }
        }
      }
      {  // WB cross rounds: QTT_JAC_UNROLL fixed-slot rounds per register rotation
        constexpr int U = (WB < QTT_JAC_UNROLL) ? WB : QTT_JAC_UNROLL;
#pragma unroll 1
        for (int u = 0; u < WB; u += U) {
          cross_rounds<RPL, WB, 0, U>(X, nrm, dsc, esc, csb, slot_col, tol, noise, rot);
          if constexpr (U < WB) rotate_Jn<RPL, WB, U>(X, slot_col);
        }
      }
      // slots are back in natural order (WB-1 circle rotations and WB J rotations = identity)
#pragma unroll
      for (int c = 0; c < WB; ++c) {
#if QTT_JAC_SCALED
        const double dI = dsc[c], dJ = dsc[WB + c];      // fold the column scales in
#else
        const double dI = 1.0, dJ = 1.0;
#endif
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          A[(size_t)(I * WB + c) * kLdA + lane + 32 * t] = X[c][t] * dI;
          A[(size_t)(J * WB + c) * kLdA + lane + 32 * t] = X[WB + c][t] * dJ;
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    if (lane == 0 && rot) atomicOr(flag, rot);
    __syncthreads();
    const int any = *flag;
    __syncthreads();
    if (!(any & 1)) { ++sweep; break; }
#if QTT_JAC_GRAMCHECK
    // Every pair of this sweep started within |cos| < 1e-6, so by the quadratic convergence of
    // cyclic Jacobi the next sweep is (almost always) the verification sweep that rotates
    // nothing.  Check that directly on the Gram matrix (DMMA, ~1/10 of a sweep) with the same
    // threshold as the sweep's own test (whose register dot products carry rounding of the
    // same ~sqrt(m) eps order); a failed check just runs the sweep.
    if (!(any & 2) && gram_converged<NW, RPL>(A, 2 * NW * WB, tol, noise, scratch, flag)) { ++sweep; break; }
#endif
  }
  if (scale != 1.0) {
    const double inv = 1.0 / scale;
    for (int idx = threadIdx.x; idx < 2 * NW * WB * 32 * RPL; idx += NW * 32)
      A[(size_t)(idx / (32 * RPL)) * kLdA + idx % (32 * RPL)] *= inv;
    __syncthreads();
  }
  return sweep;
}

// Dispatch on the padded sizes: RPL = ceil(m/32) in {1,2,4}, WB = ceil(p/(2 NW)) (powers of 2,
// 2*NW*WB <= 128 columns).  The caller zero-pads rows to 32*RPL and columns to 2*NW*WB.
template <int NW>
__device__ __forceinline__ int jacobi_dispatch(double *A, int m, int p, int *flag, double *nrm_all, bool noise_ok) {
  const int rpl = (m <= 32) ? 1 : (m <= 64) ? 2 : 4;
  const int wb = (p <= 2 * NW) ? 1 : (p <= 4 * NW) ? 2 : (p <= 8 * NW) ? 4 : 8;
#define QTT_JAC(R, W) if (rpl == R && wb == W) return jacobi_blocked<R, W, NW>(A, m, flag, nrm_all, noise_ok);
  QTT_JAC(1, 1) QTT_JAC(1, 2) QTT_JAC(1, 4)
  QTT_JAC(2, 1) QTT_JAC(2, 2) QTT_JAC(2, 4)
  QTT_JAC(4, 1) QTT_JAC(4, 2) QTT_JAC(4, 4)
  if constexpr (NW <= 8) {
    QTT_JAC(1, 8) QTT_JAC(2, 8) QTT_JAC(4, 8)
  }
#undef QTT_JAC
  return kJacobiMaxSweeps;
}

}  // namespace qtt
