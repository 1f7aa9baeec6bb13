// qr_std.cuh -- a1 of the small path ("shift their
// normalization center to the left end", "for example using a QR
// decomposition"): one site of the right-to-left orthonormalisation sweep as a blocked
// Householder QR with explicit Q, in the LAPACK dgeqrf / dorgqr structure.
//
// Core q is the r x c row-major matrix M (r = left rank <= 64, c = legs * right rank <= 128).
// A = M^T (c x r) is staged in shared memory (row stride kLdQ, rows padded to 128 with zeros);
// A = Q R with k = min(c, r) reflectors stored below the diagonal (unit diagonal implicit) and
// R in the upper triangle.  Factorisation: 8-column register panels factored by one warp with
// straight-line updates (no divergence guards between the broadcasts), the rest of the matrix
// updated in compact-WY form on DMMA (Y = V^T C, Z by the tau recurrence over G = V^T V,
// C -= V Z) by the other warps with a one-panel lookahead -- the same structure as the a3 QR in
// qr_small.cuh, for a plain (not incremental) QR.  Q (c x k) = H_0 ... H_{k-1} [I; 0] is formed
// in a second buffer by the same WY update with the blocks taken last to first.  Then
// core q <- Q^T (k x c) and the left neighbour (rows_prev x r) <- prev R^T (rows_prev x k).
#pragma once
#include "common.cuh"
#include "qr_small.cuh"

namespace qtt {

#ifndef QTT_A1_TMA
#define QTT_A1_TMA 1          // stage the left neighbour by TMA bulk copies
#endif
constexpr int kLdQm = 68;     // Q buffer row stride (== 4 mod 16: conflict-free DMMA fragments)
constexpr int kGld = 9;       // 8 x 8 panel Gram, padded

// doubles of shared memory orth_site_blk needs
// (A, Q -- later the staged left neighbour --, scratch: Y/Z + panel Gram, tau)
constexpr int kOrthScratch = 8 * kYld + 8 * kGld;
__host__ __device__ constexpr long long orth_blk_smem() {
  return (long long)kQBkDoubles + 128 * kLdQm + kOrthScratch + 2 * kSmall;
}
static_assert(8 * kYld + 8 * kGld <= kOrthScratch, "qr_std.cuh: scratch too small");

// reflector j's component in row `row` (LAPACK storage: zero above the diagonal, unit on it)
__device__ __forceinline__ double std_v(const double *A, int row, int j) {
  const double a = A[row * kLdQ + j];              // unconditional load + selects: no branches
  return row > j ? a : (row == j ? 1.0 : 0.0);
}

// Panel j0 .. j0+7 (columns < kq) of A, factored by one warp in registers.  JT = j0 / 32 is a
// template parameter: register slot t < JT holds rows above the panel (R, never touched), slot
// t > JT rows below it (always active); only slot JT needs per-row masks (rows j0 .. j0+7 hold
// the diagonal block).  A run-time slot index would also turn the registers into local memory.
template <int JT>
__device__ __forceinline__ void std_panel(double *A, double *tau, int kq, int ncol, int j0) {
  const int lane = threadIdx.x & 31;
  double P[kPanel][4];
#pragma unroll
  for (int cc = 0; cc < kPanel; ++cc)
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (t >= JT) P[cc][t] = (j0 + cc < ncol) ? A[(lane + 32 * t) * kLdQ + j0 + cc] : 0.0;
#pragma unroll
  for (int jj = 0; jj < kPanel; ++jj) {
    const int j = j0 + jj;
    if (j < kq) {                                  // warp-uniform
      const int jl = j & 31;                       // j >> 5 == JT (j0 % 32 <= 24, jj < 8)
      const bool below = lane > jl;                // slot JT: row below the diagonal
      // masked dots over the rows below the diagonal (one reduce-scatter for the norm and the
      // panel dots) and the diagonal-row values of the panel columns (one shuffle each)
      double v[kPanel];
#pragma unroll
      for (int cc = 0; cc < kPanel; ++cc) {
        double d = 0.0;
        if (cc >= jj) {
          d = (below ? P[jj][JT] : 0.0) * P[cc][JT];
#pragma unroll
          for (int t = JT + 1; t < 4; ++t) d = fma(P[jj][t], P[cc][t], d);
        }
        v[cc] = d;
      }
      double rj[kPanel];
#pragma unroll
      for (int cc = 0; cc < kPanel; ++cc) rj[cc] = (cc >= jj) ? __shfl_sync(0xffffffffu, P[cc][JT], jl) : 0.0;
      halve<kPanel, 16, kPanel>(v, lane);
      double bc[kPanel];
#pragma unroll
      for (int cc = 0; cc < kPanel; ++cc) bc[cc] = (cc >= jj) ? __shfl_sync(0xffffffffu, v[0], cc << kPanelSh) : 0.0;
      double tj, beta, scale;
      householder_fast(rj[jj], bc[jj], tj, beta, scale);
      // column jj: v below the diagonal, beta on it
      P[jj][JT] = below ? P[jj][JT] * scale : (lane == jl ? beta : P[jj][JT]);
#pragma unroll
      for (int t = JT + 1; t < 4; ++t) P[jj][t] *= scale;
      if (lane == 0) tau[j] = tj;
      // columns cc > jj: x -= tau v (v^T x), v^T x = x_j + scale * (x_j+1.. . x) (tau = 0: w = 0)
#pragma unroll
      for (int cc = 0; cc < kPanel; ++cc) {
        if (cc > jj) {                             // (jj-independent bounds: fully unrolled)
          const double w = tj * fma(scale, bc[cc], rj[cc]);
          P[cc][JT] = below ? fma(-w, P[jj][JT], P[cc][JT]) : (lane == jl ? P[cc][JT] - w : P[cc][JT]);
#pragma unroll
          for (int t = JT + 1; t < 4; ++t) P[cc][t] = fma(-w, P[jj][t], P[cc][t]);
        }
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int cc = 0; cc < kPanel; ++cc)
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (t >= JT && j0 + cc < ncol) A[(lane + 32 * t) * kLdQ + j0 + cc] = P[cc][t];
}

// C[:, cbeg:cend) <- (H_j0 ... H_jn-1)^T C (forward: H_j0 applied first; the factorisation) or
// H_j0 ... H_jn-1 C (backward; Q formation), reflectors j0..jn-1 from A, in compact-WY form:
// Y = V^T C (DMMA; with the panel Gram G = V^T V when gram), Z by the tau recurrence,
// C -= V Z (DMMA).  Rows above j0 are untouched (V is zero there).  Run by nw warps, lw the
// calling warp's index among them.
static __device__ void std_wy(const double *A, const double *tau, double *Ysm, double *Gsm, int j0, int jn,
                              double *C, int ldc, int cbeg, int cend, bool gram, bool backward, int lw, int nw) {
  const int lane = threadIdx.x & 31, warp = lw, tid = lw * 32 + lane;
  const int np = jn - j0;
  const int gr = lane >> 2, gc = lane & 3;
  const int kbeg = j0 & ~3;                      // V is zero above row j0
  // (1) Y (8 x cols) = V^T C[:, cols]; tile -1 = the Gram V^T V
  {
    const int ntile = (cend - cbeg + 7) >> 3;
    for (int nt = warp - (gram ? 1 : 0); nt < ntile; nt += nw) {
      double c0[4] = {0.0, 0.0, 0.0, 0.0}, c1[4] = {0.0, 0.0, 0.0, 0.0};
      const int bcol = (nt < 0) ? j0 + gr : cbeg + nt * 8 + gr;
      const bool bok = (nt < 0) ? gr < np : bcol < cend;
      const int ar = j0 + gr;                     // A fragment: reflector gr, row k
      const bool aok = gr < np;
      int k0 = kbeg;
      for (; k0 + 16 <= kSmall; k0 += 16) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int k = k0 + 4 * h + gc;
          const double av = aok ? std_v(A, k, ar) : 0.0;
          const double b = !bok ? 0.0 : (nt < 0 ? std_v(A, k, bcol) : C[k * ldc + bcol]);
          dmma884(c0[h], c1[h], av, b);
        }
      }
      for (; k0 < kSmall; k0 += 4) {
        const int k = k0 + gc;
        const double av = aok ? std_v(A, k, ar) : 0.0;
        const double b = !bok ? 0.0 : (nt < 0 ? std_v(A, k, bcol) : C[k * ldc + bcol]);
        dmma884(c0[0], c1[0], av, b);
      }
      const double y0 = (c0[0] + c0[1]) + (c0[2] + c0[3]), y1 = (c1[0] + c1[1]) + (c1[2] + c1[3]);
      if (nt < 0) {
        Gsm[gr * kGld + 2 * gc] = y0;
        Gsm[gr * kGld + 2 * gc + 1] = y1;
      } else {
        const int col = cbeg + nt * 8 + 2 * gc;
        if (col < cend) Ysm[gr * kYld + col] = y0;
        if (col + 1 < cend) Ysm[gr * kYld + col + 1] = y1;
      }
    }
  }
  wy_sync(nw);
  // (2) Z per column (the sequential reflector recurrence, exactly)
  for (int c = cbeg + tid; c < cend; c += nw * 32) {
    double z[kPanel];
    if (!backward) {
#pragma unroll
      for (int jj = 0; jj < kPanel; ++jj) {
        z[jj] = 0.0;
        if (jj < np) {
          double y = Ysm[jj * kYld + c];
#pragma unroll
          for (int i = 0; i < jj; ++i) y = fma(-Gsm[i * kGld + jj], z[i], y);
          z[jj] = tau[j0 + jj] * y;
        }
      }
    } else {
#pragma unroll
      for (int jj = kPanel - 1; jj >= 0; --jj) {
        z[jj] = 0.0;
        if (jj < np) {
          double y = Ysm[jj * kYld + c];
#pragma unroll
          for (int i = jj + 1; i < kPanel; ++i)
            if (i < np) y = fma(-Gsm[i * kGld + jj], z[i], y);
          z[jj] = tau[j0 + jj] * y;
        }
      }
    }
#pragma unroll
    for (int jj = 0; jj < kPanel; ++jj)
      if (jj < np) Ysm[jj * kYld + c] = z[jj];
  }
  wy_sync(nw);
  // (3) C[j0:, cols] -= V Z   (8 x 8 tiles, K = np <= 8)
  {
    constexpr int CT = QTT_QR_CT;
    const int nct = (cend - cbeg + 7) >> 3;
    for (int rt = (j0 >> 3) + warp; rt < kSmall / 8; rt += nw) {
      const int row = rt * 8 + gr;
      double af[kPanel / 4];
#pragma unroll
      for (int ks = 0; ks < kPanel / 4; ++ks) {
        const int kk = ks * 4 + gc;
        af[ks] = (kk < np) ? -std_v(A, row, j0 + kk) : 0.0;
      }
      double *crow = C + (size_t)row * ldc;
      for (int ct0 = 0; ct0 < nct; ct0 += CT) {
        double c0[CT], c1[CT], zb[CT][kPanel / 4];
#pragma unroll
        for (int u = 0; u < CT; ++u) {
          const int cb = cbeg + (ct0 + u) * 8, cc0 = cb + 2 * gc, zc = cb + gr;
          c0[u] = (cc0 < cend) ? crow[cc0] : 0.0;
          c1[u] = (cc0 + 1 < cend) ? crow[cc0 + 1] : 0.0;
#pragma unroll
          for (int ks = 0; ks < kPanel / 4; ++ks) {
            const int kk = ks * 4 + gc;
            zb[u][ks] = (kk < np && zc < cend) ? Ysm[kk * kYld + zc] : 0.0;
          }
        }
#pragma unroll
        for (int u = 0; u < CT; ++u)
#pragma unroll
          for (int ks = 0; ks < kPanel / 4; ++ks) dmma884(c0[u], c1[u], af[ks], zb[u][ks]);
#pragma unroll
        for (int u = 0; u < CT; ++u) {
          const int cc0 = cbeg + (ct0 + u) * 8 + 2 * gc;
          if (cc0 < cend) crow[cc0] = c0[u];
          if (cc0 + 1 < cend) crow[cc0 + 1] = c1[u];
        }
      }
    }
  }
  wy_sync(nw);
}

// One a1 site (see the file comment).  core: r x c row-major (global), overwritten by Q^T
// (k x c); prev: rows_prev x r (global), overwritten by prev R^T (rows_prev x k).  Requires
// c <= 128, r <= 64 and orth_blk_smem() doubles of shared memory; kST threads.  Returns k.
__device__ __forceinline__ int orth_site_blk(double *core, int c, int r, double *prev, int rows_prev, double *smem) {
  const int tid = threadIdx.x, warp = tid >> 5;
  const int k = min(c, r);
  double *A = smem;                                  // 128 x kLdQ: M^T, then reflectors + R
  double *Qm = A + kQBkDoubles;                      // 128 x kLdQm: Q; later prev staging
  double *Ysm = Qm + 128 * kLdQm;                    // 8 x kYld (Y / Z)
  double *Gsm = Ysm + 8 * kYld;                      // 8 x kGld
  double *tau = Ysm + kOrthScratch;                  // [128]
  // A = M^T: A[i][j] = M[j][i] (rows i < c; zero rows up to 128, zero columns up to the panel)
  const int ncol = ((r + kPanel - 1) / kPanel) * kPanel;
  for (int idx = tid; idx < kSmall * ncol; idx += kST) {
    const int j = idx / kSmall, i = idx % kSmall;   // coalesced along i (a row of M)
    A[i * kLdQ + j] = (i < c && j < r) ? core[(size_t)j * c + i] : 0.0;
  }
  for (int idx = tid; idx < 128 * k; idx += kST) {   // Q buffer = [I_k; 0]
    const int i = idx / k, j = idx % k;
    Qm[i * kLdQm + j] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  constexpr int PW = QTT_QR_PW;
  constexpr int IW = (QTT_QR_ISOLATE && kSW > 4) ? (PW + kSW / 2) % kSW : -1;
  constexpr int NTW = kSW - 1 - (IW >= 0 ? 1 : 0);
  const int lw = warp - (warp > PW ? 1 : 0) - (IW >= 0 && warp > IW ? 1 : 0);
#if QTT_JAC_PROFILE
  const long long op0 = clock64();
#endif
  // factorisation with a one-panel lookahead (as qr_of_TH)
  auto panel = [&](int j0p) {                        // one call site per slot instantiation
    if (j0p < 32) std_panel<0>(A, tau, k, ncol, j0p);
    else std_panel<1>(A, tau, k, ncol, j0p);           // r <= 64: j0p < 64
  };
  if (warp == PW) panel(0);
  __syncthreads();
  for (int j0 = 0; j0 < k; j0 += kPanel) {
    const int jn = min(j0 + kPanel, k);
    if (jn >= ncol) break;                           // no columns right of this panel
    const int jn2 = min(jn + kPanel, ncol);
#ifdef QTT_BLK_TRACE
    const long long tr0 = clock64();
#endif
    std_wy(A, tau, Ysm, Gsm, j0, jn, A, kLdQ, jn, jn2, true, false, warp, kSW);
#ifdef QTT_BLK_TRACE
    const long long tr1 = clock64();
#endif
    if (jn < k) {
      if (warp == PW) panel(jn);
      else if (jn2 < ncol && warp != IW) std_wy(A, tau, Ysm, Gsm, j0, jn, A, kLdQ, jn2, ncol, false, false, lw, NTW);
    } else if (jn2 < ncol) {
      std_wy(A, tau, Ysm, Gsm, j0, jn, A, kLdQ, jn2, ncol, false, false, warp, kSW);
    }
#ifdef QTT_BLK_TRACE
    const long long tr2 = clock64();
#endif
    __syncthreads();
#ifdef QTT_BLK_TRACE
    const long long tr3 = clock64();
    if ((threadIdx.x & 31) == 0 && (warp == PW || warp == 0)) {
      long long *o = QTT_BLK_TRACE + (j0 / kPanel) * 8 + (warp == PW ? 0 : 4);
      o[0] = tr1 - tr0; o[1] = tr2 - tr1; o[2] = tr3 - tr2;
    }
#endif
  }
#if QTT_JAC_PROFILE
  const long long op1 = clock64();
#endif
  // Q = H_0 ... H_{k-1} [I; 0]: blocks last to first; block b touches columns >= j0 only
  for (int j0 = ((k - 1) / kPanel) * kPanel; j0 >= 0; j0 -= kPanel) {
    const int jn = min(j0 + kPanel, k);
    std_wy(A, tau, Ysm, Gsm, j0, jn, Qm, kLdQm, j0, k, true, true, warp, kSW);
  }
#if QTT_JAC_PROFILE
  const long long op2 = clock64();
#endif
#ifdef QTT_BLK_TRACE
  const long long tq0 = clock64();
#endif
  // core q <- Q^T
  for (int idx = tid; idx < k * c; idx += kST) {
    const int kk = idx / c, i = idx % c;
    core[idx] = Qm[i * kLdQm + kk];
  }
  __syncthreads();
#if QTT_JAC_PROFILE
  const long long opa = clock64();
#endif
#ifdef QTT_BLK_TRACE
  const long long opa_t = clock64();
#endif
  // prev <- prev R^T   (rows_prev x r) (r x k); R[kk][a] = A[kk][a], a >= kk.  DMMA over 8 x 8
  // output tiles (two per warp at a time), prev staged with row stride kLdQm
  double *Ps = Qm;                                   // staging (rows_prev x r, stride kLdQm)
  const int rp8 = (rows_prev + 7) & ~7, r4 = (r + 3) & ~3;
  const bool bulk = QTT_A1_TMA && (r % 4 == 0) && ((reinterpret_cast<uintptr_t>(prev) & 15) == 0);
  if (bulk) {
    // one TMA bulk copy per row of prev (r * 8 bytes, 16-byte aligned) into the padded rows
    uint64_t *bar = reinterpret_cast<uint64_t *>(tau + 2 * kSmall - 1);
    if (tid == 0) {
      tma_mbar_init(bar);
      tma_fence_proxy();                               // Qm's generic reads/writes come first
      tma_expect_tx(bar, (uint32_t)(rows_prev * r * sizeof(double)));
    }
    __syncthreads();
    if (warp == 0)
      for (int row = tid; row < rows_prev; row += 32)
        tma_load_1d(Ps + row * kLdQm, prev + (size_t)row * r, (uint32_t)(r * sizeof(double)), bar);
    for (int i = tid; i < (rp8 - rows_prev) * r4; i += kST) Ps[(rows_prev + i / r4) * kLdQm + i % r4] = 0.0;
    tma_wait(bar, 0);
  } else {
    for (int i = tid; i < rp8 * r4; i += kST) {
      const int row = i / r4, a = i % r4;
      Ps[row * kLdQm + a] = (row < rows_prev && a < r) ? prev[(size_t)row * r + a] : 0.0;
    }
  }
  __syncthreads();
#if QTT_JAC_PROFILE
  const long long opb = clock64();
#endif
#ifdef QTT_BLK_TRACE
  const long long opb_t = clock64();
#endif
  {
    const int lane = tid & 31, gr = lane >> 2, gc = lane & 3;
    const int tm = rp8 >> 3, tn = (k + 7) >> 3, nt = tm * tn;
    // four tiles per warp at a time, K split over two accumulators: eight independent DMMA
    // chains (one chain per tile leaves the warp waiting on the DMMA latency)
    constexpr int UT = 4;
    for (int t0 = warp * UT; t0 < nt; t0 += UT * kSW) {
      double c[UT][2][2];
#pragma unroll
      for (int u = 0; u < UT; ++u) c[u][0][0] = c[u][0][1] = c[u][1][0] = c[u][1][1] = 0.0;
      int i0[UT], n0[UT];
#pragma unroll
      for (int u = 0; u < UT; ++u) { const int t = min(t0 + u, nt - 1); i0[u] = (t / tn) * 8; n0[u] = (t % tn) * 8; }
#pragma unroll 2
      for (int a0 = 0; a0 < r4; a0 += 8) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int a = a0 + 4 * h + gc;
#pragma unroll
          for (int u = 0; u < UT; ++u) {
            const double av = (a < r4) ? Ps[(i0[u] + gr) * kLdQm + a] : 0.0;
            const int kk = n0[u] + gr;
            const double bv = (kk < k && a >= kk && a < r) ? A[kk * kLdQ + a] : 0.0;
            dmma884(c[u][h][0], c[u][h][1], av, bv);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UT; ++u) {
        const int t = t0 + u;
        if (t < nt) {
          const int row = i0[u] + gr, kk = n0[u] + 2 * gc;
          if (row < rows_prev) {
            const double v0 = c[u][0][0] + c[u][1][0], v1 = c[u][0][1] + c[u][1][1];
            double *dst = prev + (size_t)row * k + kk;
            if (kk + 1 < k && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
              *reinterpret_cast<double2 *>(dst) = make_double2(v0, v1);     // whole 16-byte pieces
            } else {
              if (kk < k) dst[0] = v0;
              if (kk + 1 < k) dst[1] = v1;
            }
          }
        }
      }
    }
  }
#ifdef QTT_BLK_TRACE
  const long long tq3 = clock64();
#endif
  __syncthreads();
#ifdef QTT_BLK_TRACE
  if ((threadIdx.x & 31) == 0 && warp < 8) {
    long long *o = QTT_BLK_TRACE + 64 + warp * 8;
    o[0] = opa_t - tq0; o[1] = opb_t - opa_t; o[2] = tq3 - opb_t; o[3] = clock64() - tq3;
  }
#endif
#if QTT_JAC_PROFILE
  const long long op3 = clock64();
  if (threadIdx.x == 0 && c == 128 && r == 64) {
    atomicAdd(&g_jprof[12], (unsigned long long)(op1 - op0)); atomicAdd(&g_jprof[13], (unsigned long long)(op2 - op1));
    atomicAdd(&g_jprof[14], (unsigned long long)(op3 - op2)); atomicAdd(&g_jprof[15], 1ull);
    atomicAdd(&g_jprof[20], (unsigned long long)(opa - op2)); atomicAdd(&g_jprof[21], (unsigned long long)(opb - opa));
  }
#endif
  return k;
}

}  // namespace qtt
