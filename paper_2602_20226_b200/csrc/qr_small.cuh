// qr_small.cuh -- the small-member path's a3: R of T^H for site matrices
// with m <= 128 rows, incremental Householder over 128-column row blocks of T^H with 8-column
// register panels and a compact-WY DMMA trailing update (see qr_of_TH).  Shared by the
// persistent site kernel (zipup.cu) and the per-member kernel (complex.cu, real scalars).
#pragma once
#include "common.cuh"
#include "jacobi.cuh"

#ifndef QTT_QR_PANEL
#define QTT_QR_PANEL 8
#endif
#ifndef QTT_QR_KC
#define QTT_QR_KC 4          // interleaved K chains of the Y = V^T C tiles
#endif
#ifndef QTT_QR_CT
#define QTT_QR_CT 4          // column tiles per batch in C -= V Z
#endif

namespace qtt {

constexpr int kSmall = 128;            // max rows m (and p) of a site matrix on this path
constexpr int kRpDoubles = kSmall * (kSmall + 1) / 2;  // packed R / GEMM staging / scratch (8256)
// Row stride of the QR's row block of T^H in shared memory.  == 4 mod 16: the DMMA fragment
// loads of the trailing update (lane (gr, gc) reads rows gc, columns gr, or rows gr, columns gc)
// hit every 8-byte bank exactly twice per warp (2 wavefronts, the minimum for 256 bytes); the
// odd stride of the Jacobi matrix gives up to 4.  The same buffer holds the Jacobi matrix later.
#ifndef QTT_QR_PW
#define QTT_QR_PW (kST / 32 - 1)   // the panel warp: the highest warp id wins its SMSP's issue arbitration
#endif
#ifndef QTT_QR_OOL
#define QTT_QR_OOL 0          // 1: the panel's rare Householder path out of line
#endif
#ifndef QTT_QR_ISOLATE
#define QTT_QR_ISOLATE 1
#endif
#ifndef QTT_QR_LD
#define QTT_QR_LD 132
#endif
constexpr int kLdQ = QTT_QR_LD;
constexpr int kQBkDoubles = kSmall * (kLdQ > kLdA ? kLdQ : kLdA);

// Threads per k_sweep CTA (one CTA per SM).  256 (8 warps, <= 255 registers, one block pair
// of 2 x 8 columns per warp in the Jacobi) measured faster than 512 (16 warps, <= 128
// registers, 2 x 4 columns): 90.2k vs 102.2k site-steps/s on cfg5 -- the Jacobi round is
// bound by FP64 and MIO issue, not by latency that more warps could hide.
#ifndef QTT_SWEEP_THREADS
#define QTT_SWEEP_THREADS 256
#endif
constexpr int kST = QTT_SWEEP_THREADS;
constexpr int kSW = kST / 32;
// qr_of_TH strides by kST and waits on named barriers sized for kST threads: every kernel that
// calls it must run kST threads (k_sweep, and k_zipup<double> with kThreads)
static_assert(kST == kThreads, "qr_small.cuh assumes QTT_SWEEP_THREADS == kThreads");

// a3: R (m x m upper triangular, packed row-major in Rp) of T^H, T row-major m x n, m <= n.
// Incremental Householder over row blocks of T^H (kSmall = 128 columns of T per block):
// QR([R; block]); the reflector of column j touches R[j][j] and the block column only.
// Blocked by panels of 16 columns: warp 0 factors a panel with the 16 columns x 128 rows in
// registers (4 rows per lane, warp-wide reductions, no CTA barrier inside the panel); then
// every thread pair applies the 16 reflectors to one trailing column held in registers.
// Two CTA barriers per panel; 2 blocks for n = 256.
constexpr int kPanel = QTT_QR_PANEL;
constexpr int kPanelSh = 5 - ilog2<kPanel>();   // halve<kPanel>: lane l holds index l >> kPanelSh

__device__ __forceinline__ int rp_idx(int j, int c, int m) { return j * m - (j * (j - 1)) / 2 + (c - j); }

__device__ __forceinline__ void qr_panel(double *Rp, double *Bk, double *tau, int m, int j0) {
  const int lane = threadIdx.x & 31;
  double P[kPanel][4];
#pragma unroll
  for (int cc = 0; cc < kPanel; ++cc)
#pragma unroll
    for (int t = 0; t < 4; ++t) P[cc][t] = (j0 + cc < m) ? Bk[(lane + 32 * t) * kLdQ + j0 + cc] : 0.0;
#pragma unroll
  for (int jj = 0; jj < kPanel; ++jj) {
    const int j = j0 + jj;
    if (j < m) {                                   // warp-uniform
      // one reduce-scatter gives both ||x_j||^2 (index jj) and x_j . x_c for the remaining panel
      // columns (v_j = scale * x_j below the unit entry, so v_j . x_c = scale * x_j . x_c):
      // the norm and the dot products share one latency chain
      double v[kPanel];
#pragma unroll
      for (int cc = 0; cc < kPanel; ++cc) {
        double d = 0.0;
        if (cc >= jj) {
#pragma unroll
          for (int t = 0; t < 4; ++t) d = fma(P[jj][t], P[cc][t], d);
        }
        v[cc] = d;
      }
      // R row j (independent of the reduction: issued before it)
      const double alpha = Rp[rp_idx(j, j, m)];
      double rjc[kPanel];
#pragma unroll
      for (int cc = 0; cc < kPanel; ++cc) rjc[cc] = (cc > jj && j0 + cc < m) ? Rp[rp_idx(j, j0 + cc, m)] : 0.0;
      halve<kPanel, 16, kPanel>(v, lane);
      // every broadcast at once, unconditionally (no divergence guard between them)
      double bc[kPanel];
#pragma unroll
      for (int cc = 0; cc < kPanel; ++cc) bc[cc] = (cc >= jj) ? __shfl_sync(0xffffffffu, v[0], cc << kPanelSh) : 0.0;
      double tj, beta, scale;
      householder_fast<QTT_QR_OOL>(alpha, bc[jj], tj, beta, scale);
#pragma unroll
      for (int t = 0; t < 4; ++t) P[jj][t] *= scale;
      if (lane == 0) { Rp[rp_idx(j, j, m)] = beta; tau[j] = tj; }
      // straight-line update of the remaining panel columns: tau = 0 (zero column) gives w = 0;
      // padding columns (c >= m) are zero, so their w is 0 as well
#pragma unroll
      for (int cc = 0; cc < kPanel; ++cc) {
        if (cc > jj) {                             // (jj-independent bounds: fully unrolled)
          const double w = tj * fma(scale, bc[cc], rjc[cc]);
#pragma unroll
          for (int t = 0; t < 4; ++t) P[cc][t] = fma(-w, P[jj][t], P[cc][t]);
          if (lane == 0 && j0 + cc < m) Rp[rp_idx(j, j0 + cc, m)] = rjc[cc] - w;
        }
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int cc = 0; cc < kPanel; ++cc)
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (j0 + cc < m) Bk[(lane + 32 * t) * kLdQ + j0 + cc] = P[cc][t];
}

// Trailing update of the panel j0..jn-1 (reflectors v_jj = [e_(j0+jj) on R's row; V_B[:, jj]],
// V_B = Bk columns j0..jn-1) on the columns c in [jn, m) of [R; B], in compact-WY form without
// forming T (LAPACK dlarft):  Y = V^T C (DMMA, with G = V_B^T V_B in the same GEMM),
// Z = tau-forward substitution Z_jj = tau_jj (Y_jj - sum_{i<jj} G_{i,jj} Z_i) (the sequential
// reflector recurrence, exactly), then R_p -= Z, B -= V_B Z (DMMA).  Equivalent to applying
// H_(j0) ... H_(jn-1) one after another.
constexpr int kYld = 136;            // Y/Z row stride (== 8 mod 16: conflict-free fragment loads)

__device__ __forceinline__ void dmma884(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// Barrier over the nw warps taking part in a trailing update: the whole CTA,
// or named barrier 1 when warp 0 is busy factoring the next panel (lookahead).
__device__ __forceinline__ void wy_sync(int nw) {
  if (nw == kSW) __syncthreads();
  else asm volatile("bar.sync 1, %0;" ::"r"(nw * 32) : "memory");
}

// Update columns [cbeg, cend) of [R; B] with the panel j0..jn-1 (see above).  gram: compute
// the Gram of the panel (Y columns j0..jn-1) in the same GEMM; otherwise it is already in
// Ysm from an earlier call for this panel.  Run by nw warps only, lw = the calling warp's
// index among them (0 .. nw-1).
static __device__ void qr_trailing_wy(double *Rp, double *Bk, const double *tau, double *Ysm, int m, int j0, int jn,
                               int cbeg, int cend, bool gram, int lw, int nw) {
  const int lane = threadIdx.x & 31, warp = lw, tid = lw * 32 + lane;
  const int np = jn - j0;                         // reflectors in the panel (<= kPanel)
  const int gr = lane >> 2, gc = lane & 3;        // mma fragment coordinates
  // (1) Y (kPanel x cols) = V_B^T Bk[:, cols], cols = [j0, jn) (Gram, if asked) + [cbeg, cend);
  // the K = 128 rows are split over QTT_QR_KC interleaved accumulator chains (independent DMMA
  // dependency chains, summed at the end) so a warp's tile is not one 32-deep DMMA latency chain
  {
    constexpr int KC = QTT_QR_KC;
    const int col0 = gram ? j0 : cbeg;
    const int ntile = (cend - col0 + 7) >> 3;
    for (int nt = warp; nt < ntile; nt += nw) {
      double c[kPanel / 8][KC][2];
#pragma unroll
      for (int mt = 0; mt < kPanel / 8; ++mt)
#pragma unroll
        for (int h = 0; h < KC; ++h) c[mt][h][0] = c[mt][h][1] = 0.0;
      const int bcol = col0 + nt * 8 + gr;        // B fragment: column gr, row gc
      const bool bok = bcol < cend && (bcol < jn || bcol >= cbeg);
#pragma unroll 2
      for (int k0 = 0; k0 < kSmall; k0 += 4 * KC) {
#pragma unroll
        for (int h = 0; h < KC; ++h) {
          const double *rowp = Bk + (size_t)(k0 + 4 * h + gc) * kLdQ;
          const double b = bok ? rowp[bcol] : 0.0;
#pragma unroll
          for (int mt = 0; mt < kPanel / 8; ++mt) {
            const int ar = mt * 8 + gr;           // A fragment: row gr (reflector), col gc (k)
            const double av = (ar < np) ? rowp[j0 + ar] : 0.0;
            dmma884(c[mt][h][0], c[mt][h][1], av, b);
          }
        }
      }
#pragma unroll
      for (int mt = 0; mt < kPanel / 8; ++mt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double v = c[mt][0][e];
#pragma unroll
          for (int h = 1; h < KC; ++h) v += c[mt][h][e];
          const int col = col0 + nt * 8 + 2 * gc + e;
          if (col < cend && (col < jn || col >= cbeg)) Ysm[(mt * 8 + gr) * kYld + col] = v;
        }
    }
  }
  wy_sync(nw);
  // (2) per updated column: Z = forward substitution; R rows j0..jn-1 updated
  for (int c = cbeg + tid; c < cend; c += nw * 32) {
    double z[kPanel];
#pragma unroll
    for (int jj = 0; jj < kPanel; ++jj) {
      z[jj] = 0.0;
      if (jj < np) {
        const int j = j0 + jj;
        double y = Ysm[jj * kYld + c] + Rp[rp_idx(j, c, m)];
#pragma unroll
        for (int i = 0; i < jj; ++i) y = fma(-Ysm[i * kYld + j0 + jj], z[i], y);
        z[jj] = tau[j] * y;
        Rp[rp_idx(j, c, m)] -= z[jj];
        Ysm[jj * kYld + c] = z[jj];
      }
    }
  }
  wy_sync(nw);
  // (3) B[:, cbeg:cend] -= V_B Z      (tiles of 8 rows x 8 columns, K = np <= kPanel); a warp
  // takes QTT_QR_CT column tiles of its row tile at once: all loads, then the DMMAs, then the
  // stores (independent chains; the compiler cannot reorder smem loads past the stores itself)
  {
    constexpr int CT = QTT_QR_CT;
    const int nct = (cend - cbeg + 7) >> 3;
    for (int rt = warp; rt < kSmall / 8; rt += nw) {
      double af[kPanel / 4];                        // -V_B fragments for this row tile
#pragma unroll
      for (int ks = 0; ks < kPanel / 4; ++ks) {
        const int kk = ks * 4 + gc;
        af[ks] = (kk < np) ? -Bk[(size_t)(rt * 8 + gr) * kLdQ + j0 + kk] : 0.0;
      }
      double *crow = Bk + (size_t)(rt * 8 + gr) * kLdQ;
      for (int ct0 = 0; ct0 < nct; ct0 += CT) {
        double c0[CT], c1[CT], zb[CT][kPanel / 4];
#pragma unroll
        for (int u = 0; u < CT; ++u) {
          const int cb = cbeg + (ct0 + u) * 8, cc0 = cb + 2 * gc, zc = cb + gr;
          if (kLdQ % 2 == 0 && cc0 + 1 < cend) {    // 16-byte aligned pair (even stride, even column)
            const double2 v2 = *reinterpret_cast<const double2 *>(crow + cc0);
            c0[u] = v2.x; c1[u] = v2.y;
          } else {
            c0[u] = (cc0 < cend) ? crow[cc0] : 0.0;
            c1[u] = (cc0 + 1 < cend) ? crow[cc0 + 1] : 0.0;
          }
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
          if (kLdQ % 2 == 0 && cc0 + 1 < cend) {
            *reinterpret_cast<double2 *>(crow + cc0) = make_double2(c0[u], c1[u]);
          } else {
            if (cc0 < cend) crow[cc0] = c0[u];
            if (cc0 + 1 < cend) crow[cc0 + 1] = c1[u];
          }
        }
      }
    }
  }
  wy_sync(nw);
}

#if QTT_JAC_PROFILE
// diagnostics: cycles of warp 0 (panel / small trailing / wait) and warp 1 (big trailing / wait)
#define QTT_QP_T(v) const long long v = clock64()
#define QTT_QP_ADD(w, i, d) if (threadIdx.x == 32 * (w)) atomicAdd(&g_jprof[i], (unsigned long long)(d))
#else
#define QTT_QP_T(v)
#define QTT_QP_ADD(w, i, d)
#endif

static __device__ __noinline__ void qr_of_TH(const double *T, int m, int n, double *Rp, double *Bk, double *tau, double *Ysm) {
  const int tid = threadIdx.x, warp = tid >> 5;
  QTT_QP_T(q0);
  for (int i = tid; i < kRpDoubles; i += kST) Rp[i] = 0.0;
  for (int c0 = 0; c0 < n; c0 += kSmall) {
    const int nb = min(kSmall, n - c0);
    __syncthreads();
    QTT_QP_T(s0);
    for (int idx = tid; idx < kSmall * m; idx += kST) {
      const int j = idx / kSmall, i = idx % kSmall;    // coalesced along i (columns of T)
      Bk[i * kLdQ + j] = (i < nb) ? T[(size_t)j * n + c0 + i] : 0.0;
    }
    __syncthreads();
    QTT_QP_T(s1);
    QTT_QP_ADD(0, 4, s1 - s0);
    // one-panel lookahead: the next panel's columns are updated first (all warps), then
    // warp 0 factors it while warps 1.. update the remaining columns (named barrier 1)
    // The panel warp PW (the highest id: it wins its SMSP's issue arbitration) has its SMSP to
    // itself while it factors: its partner warp PW - 4 sits out the big trailing update, whose
    // DMMAs (16 FP64-pipe cycles each) would otherwise stall every DFMA of the panel's latency
    // chain (QTT_QR_ISOLATE=0: all other warps update)
    constexpr int PW = QTT_QR_PW;
    constexpr int IW = (QTT_QR_ISOLATE && kSW > 4) ? (PW + kSW / 2) % kSW : -1;   // idle partner
    constexpr int NTW = kSW - 1 - (IW >= 0 ? 1 : 0);                             // big-update warps
    const int lw = warp - (warp > PW ? 1 : 0) - (IW >= 0 && warp > IW ? 1 : 0);   // index among them
    if (warp == PW) qr_panel(Rp, Bk, tau, m, 0);
    __syncthreads();
    for (int j0 = 0; j0 < m; j0 += kPanel) {
      const int jn = min(j0 + kPanel, m);
      if (jn >= m) break;
      const int jn2 = min(jn + kPanel, m);
      QTT_QP_T(t0);
      qr_trailing_wy(Rp, Bk, tau, Ysm, m, j0, jn, jn, jn2, true, warp, kSW);
      QTT_QP_T(t1);
      if (warp == PW) qr_panel(Rp, Bk, tau, m, jn);
      else if (jn2 < m && warp != IW) qr_trailing_wy(Rp, Bk, tau, Ysm, m, j0, jn, jn2, m, false, lw, NTW);
      QTT_QP_T(t2);
      __syncthreads();
      QTT_QP_T(t3);
      QTT_QP_ADD(PW, 6, t1 - t0); QTT_QP_ADD(PW, 5, t2 - t1); QTT_QP_ADD(PW, 8, t3 - t2);
      QTT_QP_ADD(PW == 0 ? 1 : 0, 7, t2 - t1); QTT_QP_ADD(PW == 0 ? 1 : 0, 9, t3 - t2);
    }
  }
  QTT_QP_T(q1);
  QTT_QP_ADD(0, 10, 1); QTT_QP_ADD(0, 11, q1 - q0);
}

}  // namespace qtt
