// orth.cuh -- a1 ("shift their normalization center to the
// left end", "for example using a QR decomposition"): one site of the
// right-to-left orthonormalisation sweep with the matrix held in registers.
//
// Core q is the r x c row-major matrix M (r = left rank, c = legs * right rank).  Householder
// QR of M^T (c x r): M^T = Q R, k = min(c, r); core q <- Q^T (k x c); the left neighbour
// (rows_prev x r, row-major) <- prev R^T (rows_prev x k).
//
// Register layout: column `col` of M^T (= row `col` of M, contiguous in memory) lives in warp
// col % 8, slot col / 8; lane l holds rows l + 32 t (t < RPL).  Right-looking unblocked QR with
// a one-column lookahead: in step j every warp applies reflector j to its trailing columns,
// except that the owner of column j+1 first updates that column and forms reflector j+1, so
// one CTA barrier per column suffices.  The reflectors go to shared memory (rows < j are
// stored as zeros, row j as 1); Q is then formed column by column (Q e_kk = H_0 ... H_kk e_kk),
// every warp independently, without barriers.
#pragma once
#include "common.cuh"
#include "jacobi.cuh"

namespace qtt {

// Doubles of shared memory orth_site_reg needs (reflectors, tau, R, staged left neighbour,
// GEMM staging).
__host__ __device__ constexpr long long orth_reg_smem(int rpl, int c, int r, int rows_prev) {
  return (long long)(c < r ? c : r) * (32 * rpl) + 2 * 64 + (long long)(c < r ? c : r) * r +
         (long long)rows_prev * r + 2 * 16 * 64 + 8 * kWarps;
}

// Warp all-reduce of N partial sums (N a power of two <= 32): tot[i] = sum over lanes of v[i].
// Butterfly reduce-scatter, then the N totals go out through the warp's shared-memory slot
// buf[0..N) (one store per total, broadcast loads) instead of N 64-bit shuffles.
template <int N>
__device__ __forceinline__ void warp_allreduce_vec(double (&v)[N], double (&tot)[N], double *buf) {
  const int lane = threadIdx.x & 31;
  halve<N, 16, N>(v, lane);
  constexpr int sh = 5 - ilog2<N>();
  __syncwarp();                                    // previous readers of buf are done
  if ((lane & ((1 << sh) - 1)) == 0) buf[lane >> sh] = v[0];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < N; ++i) tot[i] = buf[i];
}

template <int RPL, int NCW>
__device__ __forceinline__ void orth_form_reflector(double (&X)[NCW][RPL], int j, int c, double *vbuf, double *taus) {
  // column j lives in this warp, slot j / kWarps; it has been updated by reflectors 0..j-1
  const int lane = threadIdx.x & 31;
  const int sj = j / kWarps, tj = j >> 5;
  constexpr int CP = 32 * RPL;
  double a = 0.0, s = 0.0;
#pragma unroll
  for (int t = 0; t < RPL; ++t) {
    const int row = lane + 32 * t;
#pragma unroll
    for (int ss = 0; ss < NCW; ++ss) {
      if (ss == sj) {
        const double x = X[ss][t];
        if (t == tj) a = x;
        if (row > j && row < c) s = fma(x, x, s);
      }
    }
  }
  s = warp_sum(s);
  const double alpha = __shfl_sync(0xffffffffu, a, j & 31);
  double tau, beta, scale;
  householder_fast(alpha, s, tau, beta, scale);
#pragma unroll
  for (int t = 0; t < RPL; ++t) {
    const int row = lane + 32 * t;
    double x = 0.0;
#pragma unroll
    for (int ss = 0; ss < NCW; ++ss)
      if (ss == sj) x = X[ss][t];
    const double v = (row > j && row < c) ? x * scale : (row == j ? 1.0 : 0.0);
    vbuf[(size_t)j * CP + row] = v;
#pragma unroll
    for (int ss = 0; ss < NCW; ++ss)
      if (ss == sj && row == j) X[ss][t] = beta;     // R[j][j]
  }
  if (lane == 0) taus[j] = tau;
}

// Apply reflector j to this warp's columns col > j (only slot `only` if only >= 0, all
// slots but -2-only if only <= -2, every slot if only == -1); FORM_Q: every column, no mask.
template <int RPL, int NCW, bool FORM_Q = false>
__device__ __forceinline__ void orth_apply(double (&X)[NCW][RPL], int j, const double *vbuf, double tau, int only,
                                           double *wbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int CP = 32 * RPL;
  double v[RPL];
#pragma unroll
  for (int t = 0; t < RPL; ++t) v[t] = vbuf[(size_t)j * CP + lane + 32 * t];
  double p[NCW], tot[NCW];
#pragma unroll
  for (int ss = 0; ss < NCW; ++ss) {
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < RPL; ++t) acc = fma(v[t], X[ss][t], acc);
    p[ss] = acc;
  }
  warp_allreduce_vec<NCW>(p, tot, wbuf);
#pragma unroll
  for (int ss = 0; ss < NCW; ++ss) {
    const int col = warp + kWarps * ss;
    bool act = FORM_Q || col > j;
    if (only >= 0) act = act && (ss == only);
    else if (only <= -2) act = act && (ss != (-2 - only));
    if (act) {
      const double w = tau * tot[ss];
#pragma unroll
      for (int t = 0; t < RPL; ++t) X[ss][t] = fma(-w, v[t], X[ss][t]);
    }
  }
}

// One a1 site.  core: r x c (row-major) in global memory, overwritten by Q^T (k x c).
// prev: rows_prev x r (row-major), overwritten by prev R^T (rows_prev x k).  Requires
// c <= 32*RPL, r <= 8*NCW and orth_reg_smem(RPL, c, r, rows_prev) doubles of smem.
// Returns k.  All threads of the CTA must call it.
template <int RPL, int NCW>
__device__ int orth_site_reg(double *core, int c, int r, double *prev, int rows_prev, double *smem) {
  constexpr int CP = 32 * RPL;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = min(c, r);
  double *vbuf = smem;                              // k x CP reflectors
  double *taus = vbuf + (size_t)k * CP;             // [<=128]
  double *Rb = taus + 2 * 64;                       // k x r, upper trapezoidal
  double *Psm = Rb + (size_t)k * r;                 // rows_prev x r
  double *gst = Psm + (size_t)rows_prev * r;        // GEMM staging (2 x 16 x 64)
  double *wbuf = gst + 2 * 16 * 64 + (threadIdx.x >> 5) * 8;   // per-warp all-reduce slot

  double X[NCW][RPL];
#pragma unroll
  for (int ss = 0; ss < NCW; ++ss) {
    const int col = warp + kWarps * ss;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int row = lane + 32 * t;
      X[ss][t] = (col < r && row < c) ? core[(size_t)col * c + row] : 0.0;
    }
  }
  for (int i = tid; i < rows_prev * r; i += kThreads) Psm[i] = prev[i];
  for (int i = tid; i < k * r; i += kThreads) Rb[i] = 0.0;
  if (warp == 0) orth_form_reflector<RPL, NCW>(X, 0, c, vbuf, taus);
  __syncthreads();
#if QTT_JAC_PROFILE
  const long long op0 = clock64();
#endif
  // The owner of column j+1 applies reflector j to that column only, forms reflector j+1 and
  // defers reflector j on its other columns to the next step (where it is not the owner), so
  // the per-step critical path is one column update + one reflector, not a full update more.
  int pend = -1, pend_slot = 0;
  for (int j = 0; j < k; ++j) {
    const double tau = taus[j];
    const int nxt = j + 1;
    if (nxt < k && warp == (nxt % kWarps)) {
      const int sn = nxt / kWarps;
      if (tau != 0.0) orth_apply<RPL, NCW>(X, j, vbuf, tau, sn, wbuf);
      orth_form_reflector<RPL, NCW>(X, nxt, c, vbuf, taus);
      pend = j; pend_slot = sn;
    } else {
      if (pend >= 0) {
        const double tp = taus[pend];
        if (tp != 0.0) orth_apply<RPL, NCW>(X, pend, vbuf, tp, -2 - pend_slot, wbuf);
        pend = -1;
      }
      if (tau != 0.0) orth_apply<RPL, NCW>(X, j, vbuf, tau, -1, wbuf);
    }
    __syncthreads();
  }
  if (pend >= 0) {                                  // owner of the last column: finish its update
    const double tp = taus[pend];
    if (tp != 0.0) orth_apply<RPL, NCW>(X, pend, vbuf, tp, -2 - pend_slot, wbuf);
  }
#if QTT_JAC_PROFILE
  const long long op1 = clock64();
#endif
  // R: column col holds R[i][col] in rows i <= min(col, k-1)
#pragma unroll
  for (int ss = 0; ss < NCW; ++ss) {
    const int col = warp + kWarps * ss;
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int row = lane + 32 * t;
      if (col < r && row < k && row <= col) Rb[(size_t)row * r + col] = X[ss][t];
    }
  }
  // Q columns (kk < k): x = e_kk, then H_{k-1} ... H_0 (H_j e_kk = e_kk for j > kk exactly)
#pragma unroll
  for (int ss = 0; ss < NCW; ++ss) {
    const int col = warp + kWarps * ss;
#pragma unroll
    for (int t = 0; t < RPL; ++t) X[ss][t] = (lane + 32 * t == col) ? 1.0 : 0.0;
  }
  const int jtop = min(k - 1, warp + kWarps * (NCW - 1));  // highest column this warp owns
  for (int j = jtop; j >= 0; --j) {
    const double tau = taus[j];
    if (tau != 0.0) orth_apply<RPL, NCW, true>(X, j, vbuf, tau, -1, wbuf);
  }
  __syncthreads();                                   // Rb complete; reflectors no longer read
#if QTT_JAC_PROFILE
  const long long op2 = clock64();
#endif
  // core q <- Q^T: row kk = column kk of Q (coalesced along rows of Q)
#pragma unroll
  for (int ss = 0; ss < NCW; ++ss) {
    const int col = warp + kWarps * ss;
    if (col < k) {
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int row = lane + 32 * t;
        if (row < c) core[(size_t)col * c + row] = X[ss][t];
      }
    }
  }
  // prev <- prev R^T   (rows_prev x r) (r x k)
  cta_gemm(rows_prev, k, r, [&](int i, int a) { return Psm[(size_t)i * r + a]; },
           [&](int a, int kk) { return Rb[(size_t)kk * r + a]; },
           [&](int i, int kk, double v) { prev[(size_t)i * k + kk] = v; }, gst);
  __syncthreads();
#if QTT_JAC_PROFILE
  const long long op3 = clock64();
  if (threadIdx.x == 0 && c == 128 && r == 64) {
    atomicAdd(&g_jprof[12], (unsigned long long)(op1 - op0)); atomicAdd(&g_jprof[13], (unsigned long long)(op2 - op1));
    atomicAdd(&g_jprof[14], (unsigned long long)(op3 - op2)); atomicAdd(&g_jprof[15], 1ull);
  }
#endif
  return k;
}

}  // namespace qtt
