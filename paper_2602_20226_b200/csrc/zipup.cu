// zipup.cu -- the zip-up hot path (§3.2).
//
// Small-member path: one CTA (256 threads, 1 per SM) owns one batch member at a time.
//   k_orth : a1 right-orthonormalisation of one operand, all sites right-to-left (Householder
//            QR with explicit Q, R absorbed into the left neighbour).
//   k_sweep: persistent: every (site, member) step: a2 contraction -> T (L2-resident scratch),
//            a3 incremental Householder QR of T^H (R in shared memory), a4 one-sided Jacobi
//            SVD on R^H in shared memory (warp-shuffle reductions, round-robin ordering),
//            a5 tail-sum truncation, a6 emit U_k and carry G = U_k^T T, a7 last site.
// All ranks live on the device (int arrays); no host synchronisation anywhere.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <string.h>
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "jacobi.cuh"
#include "large.cuh"
#include "orth.cuh"
#include "qr_small.cuh"
#include "qr_std.cuh"

#ifndef QTT_A1_BLK
#define QTT_A1_BLK 1          // a1 wide sites by the blocked QR of qr_std.cuh
#endif
#ifndef QTT_A1_BLK_MINR
#define QTT_A1_BLK_MINR 17
#endif
static_assert(qtt::orth_blk_smem() <= 27904, "a1 blocked path exceeds the k_orth shared memory");



namespace qtt {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

qtt_status_t cuda_status(cudaError_t e, const char *what) {
  set_error("CUDA error %s in %s", cudaGetErrorString(e), what);
  return QTT_ECUDA;
}


constexpr int kMaxSites = 64;
constexpr int kBkDoubles = kRpDoubles;                  // staged MPO core limit
constexpr int kSiteSmemDoubles = kRpDoubles + kQBkDoubles + kSmall + 16 + 8 + kSmall + 16 * 136;
constexpr size_t kSiteSmemBytes = kSiteSmemDoubles * sizeof(double) + (kSmall + 8) * sizeof(int);
constexpr int kOrthSmemDoubles = 27904;  // a1 staging budget (218 KB; >= orth_blk_smem())


// ======================================================================= a1: pre-pass

struct OrthArgs {
  int L, orth, shared;
  int legs[kMaxSites];
  int r0[kMaxSites + 1];
  long long off[kMaxSites + 1];       // per-member offsets (elements) of each core in dst
  const double *src[kMaxSites];       // batch-strided input cores
  double *dst; long long dst_bs;
  int *rk;                            // [B][L+1] ranks after a1
};

// Householder QR of the c x r column-major matrix Ms (ld = c) in shared memory:
// reflectors below the diagonal, R on and above it, tau[j].  LAPACK dgeqr2 order.
__device__ void smem_geqr2(double *Ms, int c, int r, double *tau, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = min(c, r);
  for (int j = 0; j < k; ++j) {
    double *cj = Ms + (size_t)j * c;
    if (warp == 0) {
      double s = 0.0;
      for (int i = j + 1 + lane; i < c; i += 32) s += cj[i] * cj[i];
      s = warp_sum(s);
      double t, beta, scale;
      householder(cj[j], s, t, beta, scale);
      for (int i = j + 1 + lane; i < c; i += 32) cj[i] *= scale;
      __syncwarp();
      if (lane == 0) { tau[j] = t; cj[j] = beta; }
    }
    __syncthreads();
    const double t = tau[j];
    if (t != 0.0) {
      for (int col = j + 1 + warp; col < r; col += kWarps) {
        double *cc = Ms + (size_t)col * c;
        double s = (lane == 0) ? cc[j] : 0.0;
        for (int i = j + 1 + lane; i < c; i += 32) s += cj[i] * cc[i];
        s = warp_sum(s) * t;
        if (lane == 0) cc[j] -= s;
        for (int i = j + 1 + lane; i < c; i += 32) cc[i] -= s * cj[i];
      }
    }
    __syncthreads();
  }
}

// Form the first k columns of Q in place from the reflectors (LAPACK dorg2r).
__device__ void smem_org2r(double *Ms, int c, int k, const double *tau) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = k - 1; j >= 0; --j) {
    double *cj = Ms + (size_t)j * c;
    const double t = tau[j];
    if (j < k - 1 && t != 0.0) {
      for (int col = j + 1 + warp; col < k; col += kWarps) {
        double *cc = Ms + (size_t)col * c;
        double s = (lane == 0) ? cc[j] : 0.0;   // v_j = 1
        for (int i = j + 1 + lane; i < c; i += 32) s += cj[i] * cc[i];
        s = warp_sum(s) * t;
        if (lane == 0) cc[j] -= s;
        for (int i = j + 1 + lane; i < c; i += 32) cc[i] -= s * cj[i];
      }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < c; i += kThreads) {
      if (i > j) cj[i] *= -t;
      else if (i == j) cj[i] = 1.0 - t;
      else cj[i] = 0.0;
    }
    __syncthreads();
  }
}

// a shared operator's ranks (row 0 of a [B][n] int array) broadcast to every member's row
__global__ void k_bcast_row(int *rows, int n, int B) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n && i < n * B) rows[i] = rows[i % n];
}

__global__ void __launch_bounds__(kThreads, 1) k_orth(OrthArgs a) {
  extern __shared__ double smem[];
  const int b = blockIdx.x, tid = threadIdx.x;
  const int L = a.L;
  double *base = a.dst + (size_t)b * a.dst_bs;
  // copy every core of member b into the workspace (inputs are never modified): 16-byte
  // accesses with eight loads in flight per thread when both sides are aligned (an element
  // loop leaves one load in flight: ~0.5 ms per cfg5 member of pure latency)
  for (int q = 0; q < L; ++q) {
    const long long n = (long long)a.r0[q] * a.legs[q] * a.r0[q + 1];
    const double *src = a.src[q] + (a.shared ? 0 : (size_t)b * n);
    double *dst = base + a.off[q];
    long long done = 0;
    if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
      const double2 *s2 = reinterpret_cast<const double2 *>(src);
      double2 *d2 = reinterpret_cast<double2 *>(dst);
      const long long n2 = n >> 1;
      constexpr int U = 8;
      long long i = tid;
      for (; i + (U - 1) * kThreads < n2; i += U * kThreads) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(s2 + i + u * kThreads);
#pragma unroll
        for (int u = 0; u < U; ++u) d2[i + u * kThreads] = v[u];
      }
      for (; i < n2; i += kThreads) d2[i] = __ldcs(s2 + i);
      done = n2 << 1;
    }
    for (long long i = done + tid; i < n; i += kThreads) dst[i] = src[i];
  }
  int *rk = a.rk + (size_t)b * (L + 1);
  for (int q = tid; q <= L; q += kThreads) rk[q] = a.r0[q];
  __syncthreads();
  if (!a.orth) return;
  double *tau = smem;                  // [kSmall*2]
  double *red = tau + 2 * kSmall;      // [16]
  double *Ms = red + 16;
  int rr = 1;                          // current right rank of core q
  for (int q = L - 1; q >= 1; --q) {
    const int r = a.r0[q];
    const int legs = a.legs[q];
    const int c = legs * rr;
    const int k = min(c, r);
    double *core = base + a.off[q];
    {  // register-resident QR (orth.cuh) when the site fits; else the shared-memory path below
      const int rows_prev = a.r0[q - 1] * a.legs[q - 1];
#if QTT_A1_BLK
      // wide sites: blocked Householder with DMMA WY updates and explicit Q (qr_std.cuh)
      if (c > 64 && c <= 128 && r >= QTT_A1_BLK_MINR && r <= 64 && rows_prev <= 128) {
        orth_site_blk(core, c, r, base + a.off[q - 1], rows_prev, smem);
        if (tid == 0) rk[q] = k;
        rr = k;
        continue;
      }
#endif
      const int rpl = (c <= 32) ? 1 : (c <= 64) ? 2 : (c <= 128) ? 4 : 0;
      const int ncw = (r <= 8) ? 1 : (r <= 16) ? 2 : (r <= 32) ? 4 : (r <= 64) ? 8 : 0;
      if (rpl && ncw && orth_reg_smem(rpl, c, r, rows_prev) <= kOrthSmemDoubles) {
        double *prev = base + a.off[q - 1];
#define QTT_ORTH(R_, N_) \
  else if (rpl == R_ && ncw == N_) orth_site_reg<R_, N_>(core, c, r, prev, rows_prev, smem);
        if (false) {}
        QTT_ORTH(1, 1) QTT_ORTH(1, 2) QTT_ORTH(1, 4) QTT_ORTH(1, 8)
        QTT_ORTH(2, 1) QTT_ORTH(2, 2) QTT_ORTH(2, 4) QTT_ORTH(2, 8)
        QTT_ORTH(4, 1) QTT_ORTH(4, 2) QTT_ORTH(4, 4) QTT_ORTH(4, 8)
#undef QTT_ORTH
        if (tid == 0) rk[q] = k;
        rr = k;
        continue;
      }
    }
    double *Rsm = Ms + (size_t)c * r;                 // k x r
    double *Psm = Rsm + (size_t)k * r;                // rows_prev x r
    // M^T (c x r, column-major): column aa = row aa of the core (contiguous)
    for (int i = tid; i < c * r; i += kThreads) Ms[i] = core[i];
    __syncthreads();
    smem_geqr2(Ms, c, r, tau, red);
    for (int i = tid; i < k * r; i += kThreads) {
      const int kk = i / r, aa = i % r;
      Rsm[i] = (aa >= kk) ? Ms[(size_t)aa * c + kk] : 0.0;
    }
    __syncthreads();
    smem_org2r(Ms, c, k, tau);
    // core q <- Q^T (k x c): row kk = column kk of Q
    for (int i = tid; i < k * c; i += kThreads) core[i] = Ms[i];
    // core q-1 <- core q-1 x_last R^T
    const int rows = a.r0[q - 1] * a.legs[q - 1];
    double *prev = base + a.off[q - 1];
    for (int i = tid; i < rows * r; i += kThreads) Psm[i] = prev[i];
    __syncthreads();
    for (int i = tid; i < rows * k; i += kThreads) {
      const int row = i / k, kk = i % k;
      double s = 0.0;
      for (int aa = kk; aa < r; ++aa) s = fma(Psm[row * r + aa], Rsm[kk * r + aa], s);
      prev[i] = s;
    }
    if (tid == 0) rk[q] = k;
    rr = k;
    __syncthreads();
  }
}

// ======================================================================= a2..a7: site step

struct SweepArgs {
  int L, B, kind, shared_op;
  int d[kMaxSites], dj[kMaxSites];       // output / contracted digit size per site
  long long xoff[kMaxSites], ooff[kMaxSites];
  double *Cq[kMaxSites];                 // output core slots (batch-strided)
  long long Cq_bs[kMaxSites];
  const double *Xo; long long Xo_bs;     // orthonormalised x cores (workspace)
  const double *Oo; long long Oo_bs;     // orthonormalised operator cores (workspace)
  const int *xr; const int *orr;         // [B][L+1] operand ranks after a1
  int *yr;                               // [B][L+1] output ranks
  double *G; long long G_bs;             // carry (chi, w, r)
  double *T; long long T_bs;             // site matrix (m x n), row-major
  double *X; long long X_bs;             // state-contraction intermediate
  int *task_counter;                     // persistent scheduler: next (site, member) task
  int *done;                             // [B] sites completed per member (acquire/release)
  double *delta2, *norm2, *sigma;
  int sigma_stride;
  int *sweeps;
  long long *cycles;                     // optional [B][L][4] clock64 per phase
  int *status;
  double eps;
  int max_rank;
};

// a2 for "ij,j->i" on DMMA, fused with the MPO epilogue (no X round trip through global):
//   X[(c,w),(j,r')] = sum_r G[(c,w),r] x_q[r,(j,r')]     (M = chi*w, K = r, N = dj*r2)
//   T[c,i,w',r']    = sum_{w,j} X[c,w,j,r'] W[w,i,j,w']
// x_q is staged in Xs (K x 136, == 8 mod 16: conflict-free B fragments), W in Ws; every warp
// takes 8-row tiles of X (8/w whole c's, since w divides 8), accumulates 8 x N with m8n8k4
// DMMA (A fragments straight from G in L2), parks the tile in its Xt slot (8 x 129) and
// forms the tile's T rows.  Requires w in {1,2,4,8}, N <= 128, padded K * 136 <= kSmall *
// kLdA, w * d * dj * w2 <= 16 * kYld.
constexpr int kXsLd = 136, kXtLd = 129;

__device__ __forceinline__ bool contract_dmma_ok(int w, int K, int N, int wsz) {
  return (w == 1 || w == 2 || w == 4 || w == 8) && N <= 128 && ((K + 3) & ~3) * kXsLd <= kSmall * kLdA &&
         wsz <= 16 * kYld;
}

__device__ void contract_dmma(const double *G, const double *Xq, const double *Oq, double *T, int chi, int w, int K,
                              int dj, int r2, int d, int w2, double *Xs, double *Xt, double *Ws) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gr = lane >> 2, gc = lane & 3;
  const int M = chi * w, N = dj * r2, wsz = w * d * dj * w2;
  const int Kp = (K + 3) & ~3;
  for (int idx = tid; idx < Kp * N; idx += kST) {          // coalesced along N
    const int k = idx / N, n = idx - k * N;
    Xs[k * kXsLd + n] = (k < K) ? Xq[(size_t)k * N + n] : 0.0;
  }
  for (int i = tid; i < wsz; i += kST) Ws[i] = Oq[i];
  __syncthreads();
  double *xt = Xt + warp * 8 * kXtLd;
  const int ntn = (N + 7) >> 3;
  const int cpt = 8 / w;                                   // c's per 8-row tile
  for (int mt = warp; mt * 8 < M; mt += kSW) {
    double acc[16][2];
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
    const int arow = mt * 8 + gr;
    const double *ga = G + (size_t)arow * K;
    for (int k0 = 0; k0 < Kp; k0 += 4) {
      const int k = k0 + gc;
      const double av = (arow < M && k < K) ? ga[k] : 0.0;
      const double *xb = Xs + k * kXsLd + gr;
#pragma unroll
      for (int nt = 0; nt < 16; ++nt)
        if (nt < ntn) dmma884(acc[nt][0], acc[nt][1], av, xb[nt * 8]);
    }
#pragma unroll
    for (int nt = 0; nt < 16; ++nt)
      if (nt < ntn) {
        xt[gr * kXtLd + nt * 8 + 2 * gc] = acc[nt][0];
        xt[gr * kXtLd + nt * 8 + 2 * gc + 1] = acc[nt][1];
      }
    __syncwarp();
    // T rows of this tile's c's: lane -> r' (strided), loop (i, w') and (w, j)
    for (int cl = 0; cl < cpt; ++cl) {
      const int c = mt * cpt + cl;
      if (c >= chi) break;
      const double *xr = xt + cl * w * kXtLd;
      for (int rr = lane; rr < r2; rr += 32) {
        for (int ii = 0; ii < d; ++ii)
          for (int w2i = 0; w2i < w2; ++w2i) {
            double sacc = 0.0;
            for (int ww = 0; ww < w; ++ww)
              for (int jj = 0; jj < dj; ++jj)
                sacc = fma(xr[ww * kXtLd + jj * r2 + rr], Ws[((ww * d + ii) * dj + jj) * w2 + w2i], sacc);
            T[((size_t)(c * d + ii) * w2 + w2i) * r2 + rr] = sacc;
          }
      }
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void site_step(const SweepArgs &a, int b, int q, double *smem) {
  double *Rp = smem;                         // packed R (QR) / GEMM staging / scratch
  double *Rs = Rp + kRpDoubles;              // kSmall x kLdA: QR block, then A (col-major)
  double *Bk = Rp;                           // staging alias
  double *sg = Rs + kQBkDoubles;           // sigma^2 per column
  double *red = sg + kSmall;                 // block-reduction scratch
  double *scal = red + 16;                   // scalars
  double *tau = scal + 8;                    // Householder tau per column
  double *Ysm = tau + kSmall;                  // QR trailing update: Y / Z (16 x kYld)
  int *perm = reinterpret_cast<int *>(Ysm + 16 * kYld);
  int *iflag = perm + kSmall;

  const int tid = threadIdx.x;
  const int L = a.L, L1 = L + 1;
  const int chi = (q == 0) ? 1 : a.yr[(size_t)b * L1 + q];
  const int r = a.xr[(size_t)b * L1 + q], r2 = a.xr[(size_t)b * L1 + q + 1];
  int w = 1, w2 = 1;
  if (a.kind != TRUNCATE) { w = a.orr[(size_t)b * L1 + q]; w2 = a.orr[(size_t)b * L1 + q + 1]; }
  const int d = a.d[q], dj = a.dj[q];
  const int m = chi * d, n = w2 * r2;
  double *G = a.G + (size_t)b * a.G_bs;
  // T and X live only inside one task: one slot per CTA (grid <= B), so the ~148 slots in use
  // stay L2-resident and are rewritten in place instead of walking a B-slot footprint
  // (per-member slots made the dirty lines of finished tasks get written back to HBM)
#ifndef QTT_CTA_SCRATCH
#define QTT_CTA_SCRATCH 1
#endif
  const size_t slot = QTT_CTA_SCRATCH ? (size_t)blockIdx.x : (size_t)b;
  double *T = a.T + slot * a.T_bs;
  double *X = a.X + slot * a.X_bs;
  const double *Xq = a.Xo + (size_t)b * a.Xo_bs + a.xoff[q];
  const double *Oq = a.Oo ? a.Oo + (a.shared_op ? 0 : (size_t)b * a.Oo_bs) + a.ooff[q] : nullptr;
  double *Cq = a.Cq[q] + (size_t)b * a.Cq_bs[q];

  long long t_phase = clock64();
  if (q == 0) {
    if (tid == 0) G[0] = 1.0;                // G_0 = [[[1]]]
    __syncthreads();
  }
  // ---------------------------------------------------------------- a2: contraction
  if (a.kind == MATVEC && kSW == 8 && contract_dmma_ok(w, r, dj * r2, w * d * dj * w2)) {
    contract_dmma(G, Xq, Oq, T, chi, w, r, dj, r2, d, w2, Rs, Rp, Ysm);
  } else if (a.kind == MATVEC) {
    const int M = chi * w, K = r, N = dj * r2;     // X[(c,w),(j,r')] = G[(c,w),r] x_q[r,(j,r')]
    cta_gemm<kST>(M, N, K, [&](int i, int k) { return G[(size_t)i * K + k]; },
             [&](int k, int j) { return Xq[(size_t)k * N + j]; },
             [&](int i, int j, double v) { X[(size_t)i * N + j] = v; }, Bk);
    __syncthreads();
    const int wsz = w * d * dj * w2;
    for (int i = tid; i < wsz; i += kST) Bk[i] = Oq[i];
    __syncthreads();
    // T[c,i,w',r'] = sum_{w,j} X[c,w,j,r'] W[w,i,j,w']
    const int dw = d * w2;
    if (dw <= 16) {
      // one thread per (c, r'): every X value is loaded once (coalesced along r') and feeds all
      // d*w' outputs of that (c, r'); W is read from shared memory (warp-uniform addresses)
      int woff[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) woff[e] = (e < dw) ? (e / w2) * dj * w2 + e % w2 : 0;
      for (int pr = tid; pr < chi * r2; pr += kST) {
        const int c = pr / r2, rr2 = pr - c * r2;
        double acc[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) acc[e] = 0.0;
        for (int ww = 0; ww < w; ++ww)
          for (int jj = 0; jj < dj; ++jj) {
            const double xv = X[((size_t)(c * w + ww) * dj + jj) * r2 + rr2];
            const double *wr = Bk + (ww * d * dj + jj) * w2;
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (e < dw) acc[e] = fma(xv, wr[woff[e]], acc[e]);
          }
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (e < dw) T[((size_t)c * dw + e) * r2 + rr2] = acc[e];
      }
    } else
    for (int idx = tid; idx < m * n; idx += kST) {
      const int rr2 = idx % r2;
      int t1 = idx / r2;
      const int ww2 = t1 % w2; t1 /= w2;
      const int ii = t1 % d, c = t1 / d;
      double s = 0.0;
      for (int ww = 0; ww < w; ++ww)
        for (int jj = 0; jj < dj; ++jj)
          s = fma(X[((size_t)(c * w + ww) * dj + jj) * r2 + rr2], Bk[((ww * d + ii) * dj + jj) * w2 + ww2], s);
      T[idx] = s;
    }
  } else if (a.kind == HADAMARD) {
    const int M = chi * w, K = r, N = d * r2;      // X[(c,a),(i,b')] = G[(c,a),b] x_q[b,(i,b')]
    cta_gemm<kST>(M, N, K, [&](int i, int k) { return G[(size_t)i * K + k]; },
             [&](int k, int j) { return Xq[(size_t)k * N + j]; },
             [&](int i, int j, double v) { X[(size_t)i * N + j] = v; }, Bk);
    __syncthreads();
    for (int ci = 0; ci < chi * d; ++ci) {         // T[c,i,a',b'] = sum_a A[a,i,a'] X[c,a,i,b']
      const int c = ci / d, ii = ci % d;
      cta_gemm<kST>(w2, r2, w, [&](int a2, int aa) { return Oq[((size_t)aa * d + ii) * w2 + a2]; },
               [&](int aa, int bb) { return X[((size_t)(c * w + aa) * d + ii) * r2 + bb]; },
               [&](int a2, int bb, double v) { T[((size_t)(c * d + ii) * w2 + a2) * r2 + bb] = v; }, Bk);
    }
  } else {
    const int M = chi, K = r, N = d * r2;          // T[c,(i,r')] = G[c,r] x_q[r,(i,r')]
    cta_gemm<kST>(M, N, K, [&](int i, int k) { return G[(size_t)i * K + k]; },
             [&](int k, int j) { return Xq[(size_t)k * N + j]; },
             [&](int i, int j, double v) { T[(size_t)i * N + j] = v; }, Bk);
  }
  __syncthreads();
  if (tid == 0 && a.cycles) a.cycles[((size_t)b * L + q) * 4 + 0] = clock64() - t_phase;
  t_phase = clock64();

  // ---------------------------------------------------------------- a7: last site
  if (q == L - 1) {
    double s = 0.0;
    for (int i = tid; i < m; i += kST) { const double v = T[i]; Cq[i] = v; s = fma(v, v, s); }
    s = block_sum<kSW>(s, red);
    if (tid == 0) {
      if (a.sweeps) a.sweeps[(size_t)b * L + q] = 0;
      a.norm2[b] = s;
      a.delta2[(size_t)b * L + q] = 0.0;
      a.yr[(size_t)b * L1 + L] = 1;
      if (L == 1) a.yr[(size_t)b * L1] = 1;
      if (!isfinite(s)) atomicOr(a.status, ST_NONFINITE);
    }
    return;
  }

  // ---------------------------------------------------------------- a3: QR
  int p;
  if (m <= n) {
    p = m;
    qr_of_TH(T, m, n, Rp, Rs, tau, Ysm);
    __syncthreads();
    for (int idx = tid; idx < m * m; idx += kST) {   // A = R^T: column j of A = row j of R
      const int j = idx / m, row = idx % m;
      Rs[(size_t)j * kLdA + row] = (row >= j) ? Rp[rp_idx(j, row, m)] : 0.0;
    }
  } else {
    p = n;                                         // A = T (m x n): column j = T[:, j]
    for (int idx = tid; idx < m * n; idx += kST) {
      const int row = idx / n, j = idx % n;
      Rs[(size_t)j * kLdA + row] = T[idx];
    }
  }
  __syncthreads();
  if (tid == 0 && a.cycles) a.cycles[((size_t)b * L + q) * 4 + 1] = clock64() - t_phase;
  t_phase = clock64();

  // ---------------------------------------------------------------- a4: Jacobi SVD
  {  // zero padding required by the register-blocked Jacobi: rows [m, 32*RPL), columns [p, 16*WB)
    const int mp = (m <= 32) ? 32 : (m <= 64) ? 64 : 128;
    const int wbp = (p <= 2 * kSW) ? 1 : (p <= 4 * kSW) ? 2 : (p <= 8 * kSW) ? 4 : 8;
    const int pp = 2 * kSW * wbp;                   // columns the Jacobi blocks cover
    for (int idx = tid; idx < pp * mp; idx += kST) {
      const int j = idx / mp, row = idx % mp;
      if (row >= m || j >= p) Rs[(size_t)j * kLdA + row] = 0.0;
    }
    __syncthreads();
  }
  const int sweeps = jacobi_dispatch<kSW>(Rs, m, p, iflag, Bk, noise_ok(a.eps, p));   // Bk: per-warp norm scratch
  if (tid == 0 && a.cycles) a.cycles[((size_t)b * L + q) * 4 + 2] = clock64() - t_phase;
  t_phase = clock64();
  const int lane = tid & 31, warp = tid >> 5;
  for (int j = warp; j < p; j += kSW) {
    double s = 0.0;
    for (int row = lane; row < m; row += 32) { const double v = Rs[(size_t)j * kLdA + row]; s = fma(v, v, s); }
    s = warp_sum(s);
    if (lane == 0) {
      if (!isfinite(s)) { atomicOr(a.status, ST_NONFINITE); s = 0.0; }   // keep the sort well-defined
      sg[j] = s;
    }
  }
  __syncthreads();
  for (int j = tid; j < p; j += kST) {         // descending order, ties by index
    const double sj = sg[j];
    int rank = 0;
    for (int l = 0; l < p; ++l) rank += (sg[l] > sj) || (sg[l] == sj && l < j);
    perm[rank] = j;
  }
  __syncthreads();

  // ---------------------------------------------------------------- a5: truncation rule
  if (tid == 0) {
    double *tail = Bk;                             // tail[k] = sum_{j>=k} s_j^2, smallest first
    double acc = 0.0;
    tail[p] = 0.0;
    for (int jj = p - 1; jj >= 0; --jj) { acc += sg[perm[jj]]; tail[jj] = acc; }
    const double tot = acc;
    int k = p;
    const double tau = a.eps * a.eps * tot;
    for (int kk = 1; kk <= p; ++kk)
      if (tail[kk] <= tau) { k = kk; break; }
    if (a.max_rank > 0) k = min(k, a.max_rank);
    if (tot == 0.0) k = 1;
    k = max(k, 1);
    scal[1] = (double)k;
    scal[2] = tail[k];
    if (!isfinite(tot)) atomicOr(a.status, ST_NONFINITE);
    if (sweeps >= kJacobiMaxSweeps) atomicOr(a.status, ST_NOCONV);
  }
  __syncthreads();
  const int k = (int)scal[1];

  // ---------------------------------------------------------------- a6: emit + carry
  for (int idx = tid; idx < k * m; idx += kST) {   // normalise kept columns: U = A V / sigma
    const int kk = idx / m, row = idx % m;
    const int j = perm[kk];
    const double s2 = sg[j];
    double *col = Rs + (size_t)j * kLdA;
    col[row] = (s2 > 0.0) ? col[row] / sqrt(s2) : (row == kk ? 1.0 : 0.0);
  }
  __syncthreads();
  for (int idx = tid; idx < m * k; idx += kST) {   // C_q = U[:, :k] as (chi, d, k)
    const int row = idx / k, kk = idx % k;
    Cq[idx] = Rs[(size_t)perm[kk] * kLdA + row];
  }
  if (a.sigma) {
    double *sgo = a.sigma + ((size_t)b * (L - 1) + q) * a.sigma_stride;
    for (int jj = tid; jj < a.sigma_stride; jj += kST) sgo[jj] = (jj < p) ? sqrt(sg[perm[jj]]) : 0.0;
  }
  if (tid == 0) {
    if (a.sweeps) a.sweeps[(size_t)b * L + q] = sweeps;
    a.yr[(size_t)b * L1 + q + 1] = k;
    if (q == 0) a.yr[(size_t)b * L1] = 1;
    a.delta2[(size_t)b * L + q] = scal[2];
  }
  // G_{q+1}[kk][col] = sum_row U[row][kk] T[row][col]   (k x n) = diag(s_k) V_k^H
  cta_gemm<kST>(k, n, m, [&](int kk, int row) { return Rs[(size_t)perm[kk] * kLdA + row]; },
           [&](int row, int col) { return T[(size_t)row * n + col]; },
           [&](int kk, int col, double v) { G[(size_t)kk * n + col] = v; }, Bk);
  if (tid == 0 && a.cycles) a.cycles[((size_t)b * L + q) * 4 + 3] = clock64() - t_phase;
}

// Persistent sweep: one CTA per SM pulls tasks t = q*B + b (site-major, i.e. topological
// order) from a global counter.  Task (b, q) waits for member b's site q-1 (release/acquire
// on done[b]); the holder of that task was scheduled earlier and is running or finished, so
// the wait cannot deadlock.  Balances the B*L site steps over the SMs (no wave tail).
__global__ void __launch_bounds__(kST, 1) k_sweep(SweepArgs a) {
  extern __shared__ double smem[];
  __shared__ int s_task;
  const int total = a.B * a.L;
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(a.task_counter, 1);
    __syncthreads();
    const int task = s_task;
    if (task >= total) break;
    const int q = task / a.B, b = task % a.B;
    if (threadIdx.x == 0 && q > 0) {
      int v;
      long long spins = 0;
      do {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(a.done + b) : "memory");
        if (v < q) __nanosleep(64);
        if (++spins > (1LL << 28)) __trap();   // predecessor never finished: fail loudly
      } while (v < q);
      __threadfence();          // also invalidates this SM's L1: no stale carry / scratch lines
    }
    __syncthreads();
    site_step(a, b, q, smem);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.b32 [%0], %1;" :: "l"(a.done + b), "r"(q + 1) : "memory");
    }
  }
}

// ======================================================================= host side

static int parse_kind(const char *s, const qtt_trains_t *op) {
  if (s == nullptr || strcmp(s, "i->i") == 0) return op ? -1 : TRUNCATE;
  if (strcmp(s, "ij,j->i") == 0) return MATVEC;
  if (strcmp(s, "i,i->i") == 0) return HADAMARD;
  return -2;
}

static long long round4(long long v) { return (v + 3) & ~3LL; }

static qtt_status_t analyse(const char *subs, const qtt_trains_t *op, const qtt_trains_t *x,
                           int32_t max_rank, Shape &S) {
  if (!x) { set_error("x is NULL"); return QTT_EINVAL; }
  const int kind = parse_kind(subs, op);
  if (kind == -2) { set_error("unsupported subscripts '%s'", subs); return QTT_EUNSUPPORTED; }
  if (kind == -1) { set_error("subscripts 'i->i' take no operator"); return QTT_EINVAL; }
  if (kind != TRUNCATE && !op) { set_error("operator is NULL"); return QTT_EINVAL; }
  const int L = x->n_sites;
  if (L < 1 || L > kMaxSites) { set_error("n_sites %d outside [1,%d]", L, kMaxSites); return QTT_EUNSUPPORTED; }
  if (x->n_legs != 1) { set_error("x must be an MPS (n_legs 1)"); return QTT_ESHAPE; }
  if (x->batch < 1) { set_error("batch < 1"); return QTT_EINVAL; }
  if (!x->d_out || !x->ranks || !x->cores) { set_error("x has NULL arrays"); return QTT_EINVAL; }
  if (x->ranks[0] != 1 || x->ranks[L] != 1) { set_error("x boundary ranks must be 1"); return QTT_ESHAPE; }
  S.L = L; S.B = x->batch; S.kind = kind;
  S.d.assign(L, 0); S.dj.assign(L, 0);
  S.xr.assign(x->ranks, x->ranks + L + 1);
  S.orr.assign(L + 1, 1);
  for (int q = 0; q < L; ++q) {
    if (x->d_out[q] < 1 || x->ranks[q + 1] < 1) { set_error("x site %d: bad extent", q); return QTT_ESHAPE; }
  }
  if (kind != TRUNCATE) {
    if (op->n_sites != L) { set_error("operator has %d sites, x has %d", op->n_sites, L); return QTT_ECONFORM; }
    if (op->batch != 1 && op->batch != x->batch) { set_error("operator batch must be 1 or x batch"); return QTT_EINVAL; }
    if (!op->d_out || !op->ranks || !op->cores) { set_error("operator has NULL arrays"); return QTT_EINVAL; }
    if (op->ranks[0] != 1 || op->ranks[L] != 1) { set_error("operator boundary ranks must be 1"); return QTT_ESHAPE; }
    S.shared_op = (op->batch == 1 && x->batch > 1);
    S.orr.assign(op->ranks, op->ranks + L + 1);
    if (kind == MATVEC) {
      if (op->n_legs != 2 || !op->d_in) { set_error("'ij,j->i' needs an MPO operator"); return QTT_ESHAPE; }
      for (int q = 0; q < L; ++q) {
        if (op->d_in[q] != x->d_out[q]) {
          set_error("conformance: letter 'j' misaligned at core %d (%d vs %d)", q, op->d_in[q], x->d_out[q]);
          return QTT_ECONFORM;
        }
        S.d[q] = op->d_out[q]; S.dj[q] = op->d_in[q];
      }
    } else {
      if (op->n_legs != 1) { set_error("'i,i->i' needs two MPS operands"); return QTT_ESHAPE; }
      for (int q = 0; q < L; ++q) {
        if (op->d_out[q] != x->d_out[q]) {
          set_error("conformance: letter 'i' misaligned at core %d (%d vs %d)", q, op->d_out[q], x->d_out[q]);
          return QTT_ECONFORM;
        }
        S.d[q] = S.dj[q] = x->d_out[q];
      }
    }
  } else {
    for (int q = 0; q < L; ++q) S.d[q] = S.dj[q] = x->d_out[q];
  }
  // capacities
  S.cap.assign(L + 1, 1);
  for (int q = 0; q < L; ++q) {
    long long c = (long long)S.cap[q] * S.d[q];
    c = std::min<long long>(c, (long long)S.orr[q + 1] * S.xr[q + 1]);
    if (max_rank > 0) c = std::min<long long>(c, max_rank);
    S.cap[q + 1] = (q == L - 1) ? 1 : (int)c;
  }
  // workspace geometry (per member, elements)
  S.xoff.assign(L + 1, 0); S.ooff.assign(L + 1, 0);
  for (int q = 0; q < L; ++q) {
    S.xoff[q + 1] = S.xoff[q] + (long long)S.xr[q] * S.dj[q] * S.xr[q + 1];
    long long oe = 0;
    if (kind == MATVEC) oe = (long long)S.orr[q] * S.d[q] * S.dj[q] * S.orr[q + 1];
    else if (kind == HADAMARD) oe = (long long)S.orr[q] * S.d[q] * S.orr[q + 1];
    S.ooff[q + 1] = S.ooff[q] + oe;
  }
  S.xo_elems = round4(S.xoff[L]);
  S.oo_elems = round4(S.ooff[L]);
  for (int q = 0; q < L; ++q) {
    const long long m = (long long)S.cap[q] * S.d[q];
    const long long n = (long long)S.orr[q + 1] * S.xr[q + 1];
    S.g_elems = std::max(S.g_elems, (long long)S.cap[q] * S.orr[q] * S.xr[q]);
    S.g_elems = std::max(S.g_elems, (long long)S.cap[q + 1] * n);
    S.t_elems = std::max(S.t_elems, m * n);
    if (kind == MATVEC) S.x_elems = std::max(S.x_elems, (long long)S.cap[q] * S.orr[q] * S.dj[q] * S.xr[q + 1]);
    if (kind == HADAMARD) S.x_elems = std::max(S.x_elems, (long long)S.cap[q] * S.orr[q] * S.d[q] * S.xr[q + 1]);
  }
  S.g_elems = round4(S.g_elems); S.t_elems = round4(S.t_elems); S.x_elems = round4(S.x_elems);
  return QTT_OK;
}

static qtt_status_t check_small_path(const Shape &S) {
  auto a1_ok = [&](void) { return a1_fits(S, true) ? QTT_OK : QTT_EUNSUPPORTED; };
  for (int q = 0; q < S.L; ++q) {
    const long long m = (long long)S.cap[q] * S.d[q];
    if (m > kSmall) {
      set_error("site %d: site matrix has %lld rows > %d (large-member path not in this build)", q, m, kSmall);
      return QTT_EUNSUPPORTED;
    }
    if (S.kind == MATVEC && (long long)S.orr[q] * S.d[q] * S.dj[q] * S.orr[q + 1] > kBkDoubles) {
      set_error("site %d: operator core too large to stage", q);
      return QTT_EUNSUPPORTED;
    }
  }
  return a1_ok();
}

// a1 staging budget of k_orth's shared-memory QR for both operands (x, and the operator unless
// truncating): false when some core's (c x r) block + R + the previous core exceed
// kOrthSmemDoubles or r > 2 kSmall.  report: set the thread-local error message.
bool a1_fits(const Shape &S, bool report) {
  for (int pass = 0; pass < 2; ++pass) {
    const std::vector<int> &rk = pass == 0 ? S.xr : S.orr;
    if (pass == 1 && S.kind == TRUNCATE) break;
    int rr = 1;
    for (int q = S.L - 1; q >= 1; --q) {
      const int legs = (pass == 0) ? S.dj[q] : (S.kind == MATVEC ? S.d[q] * S.dj[q] : S.d[q]);
      const int legsp = (pass == 0) ? S.dj[q - 1] : (S.kind == MATVEC ? S.d[q - 1] * S.dj[q - 1] : S.d[q - 1]);
      const long long c = (long long)legs * rr, r = rk[q], k = std::min<long long>(c, r);
      const long long need = 2 * kSmall + 16 + c * r + k * r + (long long)rk[q - 1] * legsp * r;
      if (need > kOrthSmemDoubles || r > 2 * kSmall) {
        if (report)
          set_error("a1: core %d of operand %d too large for the shared-memory QR (%lld doubles)", q, pass, need);
        return false;
      }
      rr = (int)k;
    }
  }
  return true;
}

struct WsLayout {
  size_t xo, oo, g, t, x, xr, orr, sched, total;
};

static WsLayout layout(const Shape &S) {
  WsLayout w;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  w.xo = take(sizeof(double) * S.xo_elems * S.B);
  w.oo = take(sizeof(double) * S.oo_elems * (S.shared_op ? 1 : S.B));
  w.g = take(sizeof(double) * S.g_elems * S.B);
  w.t = take(sizeof(double) * S.t_elems * S.B);
  w.x = take(sizeof(double) * S.x_elems * S.B);
  w.xr = take(sizeof(int) * (S.L + 1) * S.B);
  w.orr = take(sizeof(int) * (S.L + 1) * S.B);
  w.sched = take(sizeof(int) * (1 + S.B));
  w.total = off;
  return w;
}

// ======================================================================= fp32 variant

constexpr uint32_t kFlagTF32 = 1u << 30;     // internal: large-path contraction GEMMs as 3xTF32

struct CvtArgs {
  int L;
  const void *src[kMaxSites];
  void *dst[kMaxSites];
  long long n[kMaxSites];
};

// binary32 <-> binary64 copies of every core of one train (blockIdx.y = site)
template <bool TO64>
__global__ void k_cvt(CvtArgs a) {
  const int q = blockIdx.y;
  if (q >= a.L) return;
  const long long n = a.n[q];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (TO64) static_cast<double *>(a.dst[q])[i] = (double)static_cast<const float *>(a.src[q])[i];
    else static_cast<float *>(a.dst[q])[i] = (float)static_cast<const double *>(a.src[q])[i];
  }
}

static long long train_elems(const qtt_trains_t *t, int q) {
  return (long long)t->batch * t->ranks[q] * t->d_out[q] * (t->n_legs == 2 ? t->d_in[q] : 1) * t->ranks[q + 1];
}

// fp64 views of (op, x, out) carved from the front of the workspace
struct F32Stage {
  std::vector<void *> xp, op, outp;
  qtt_trains_t x64{}, op64{}, out64{};
  size_t bytes = 0;
};

static void f32_stage(const qtt_trains_t *op, const qtt_trains_t *x, const qtt_trains_t *out, char *ws, F32Stage &F) {
  size_t off = 0;
  auto take = [&](long long n) { void *p = ws ? (void *)(ws + off) : nullptr; off += ((size_t)n * 8 + 255) & ~size_t(255); return p; };
  const int L = x->n_sites;
  F.xp.resize(L); F.outp.resize(L);
  for (int q = 0; q < L; ++q) F.xp[q] = take(train_elems(x, q));
  if (op) { F.op.resize(L); for (int q = 0; q < L; ++q) F.op[q] = take(train_elems(op, q)); }
  if (out) for (int q = 0; q < L; ++q) F.outp[q] = take(train_elems(out, q));
  F.x64 = *x; F.x64.cores = F.xp.data(); F.x64.dtype = QTT_F64;
  if (op) { F.op64 = *op; F.op64.cores = F.op.data(); F.op64.dtype = QTT_F64; }
  if (out) { F.out64 = *out; F.out64.cores = F.outp.data(); F.out64.dtype = QTT_F64; }
  F.bytes = off;
}

static qtt_status_t cvt_train(const qtt_trains_t *t, void *const *src, void *const *dst, bool to64, cudaStream_t s) {
  CvtArgs a;
  memset(&a, 0, sizeof(a));
  a.L = t->n_sites;
  long long mx = 1;
  for (int q = 0; q < a.L; ++q) { a.src[q] = src[q]; a.dst[q] = dst[q]; a.n[q] = train_elems(t, q); mx = std::max(mx, a.n[q]); }
  dim3 grid((unsigned)std::min<long long>((mx + 255) / 256, 1024), (unsigned)a.L);
  if (to64) k_cvt<true><<<grid, 256, 0, s>>>(a);
  else k_cvt<false><<<grid, 256, 0, s>>>(a);
  QTT_CUDA_TRY(cudaGetLastError());
  return QTT_OK;
}

// -1: mixed (error), 0: fp64, 1: fp32, 2: complex128
static int train_dtypes(const qtt_trains_t *op, const qtt_trains_t *x, const qtt_trains_t *out) {
  const int dx = x ? x->dtype : QTT_F64;
  const int dop = op ? op->dtype : dx, dout = out ? out->dtype : dx;
  if (dx == QTT_F64 && dop == QTT_F64 && dout == QTT_F64) return 0;
  if (dx == QTT_F32 && dop == QTT_F32 && dout == QTT_F32) return 1;
  if (dx == QTT_C128 && dop == QTT_C128 && dout == QTT_C128) return 2;
  return -1;
}

// a1 of the fp64 path (k_orth, register-resident Householder) for the per-member kernel:
// member b's orthonormalised x cores go to xdst + b * dst_bs (+ S.xoff[q]), the operator's to
// odst + b * dst_bs (+ S.ooff[q]; a shared operator only to member 0's slot), ranks to
// xr_out / orr_out [B][L+1] (a shared operator's ranks are broadcast).
qtt_status_t orth_prepass(const Shape &S, const qtt_trains_t *op, const qtt_trains_t *x, uint32_t flags, double *xdst,
                          double *odst, long long dst_bs, int *xr_out, int *orr_out, cudaStream_t s) {
  QTT_CUDA_TRY(cudaFuncSetAttribute(k_orth, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(kOrthSmemDoubles * sizeof(double))));
  {
    OrthArgs oa;
    memset(&oa, 0, sizeof(oa));
    oa.L = S.L; oa.orth = 1; oa.shared = 0;
    for (int q = 0; q < S.L; ++q) { oa.legs[q] = S.dj[q]; oa.src[q] = (const double *)x->cores[q]; oa.off[q] = S.xoff[q]; }
    for (int q = 0; q <= S.L; ++q) oa.r0[q] = S.xr[q];
    oa.dst = xdst; oa.dst_bs = dst_bs; oa.rk = xr_out;
    k_orth<<<S.B, kThreads, kOrthSmemDoubles * sizeof(double), s>>>(oa);
    QTT_CUDA_TRY(cudaGetLastError());
  }
  if (S.kind != TRUNCATE) {
    OrthArgs oa;
    memset(&oa, 0, sizeof(oa));
    oa.L = S.L; oa.orth = (flags & QTT_NO_OPERATOR_ORTH) ? 0 : 1; oa.shared = S.shared_op;
    for (int q = 0; q < S.L; ++q) {
      oa.legs[q] = (S.kind == MATVEC) ? S.d[q] * S.dj[q] : S.d[q];
      oa.src[q] = (const double *)op->cores[q];
      oa.off[q] = S.ooff[q];
    }
    for (int q = 0; q <= S.L; ++q) oa.r0[q] = S.orr[q];
    oa.dst = odst; oa.dst_bs = dst_bs; oa.rk = orr_out;
    const int nb = S.shared_op ? 1 : S.B;
    k_orth<<<nb, kThreads, kOrthSmemDoubles * sizeof(double), s>>>(oa);
    QTT_CUDA_TRY(cudaGetLastError());
    if (S.shared_op && S.B > 1) {
      k_bcast_row<<<(S.B * (S.L + 1) + 255) / 256, 256, 0, s>>>(orr_out, S.L + 1, S.B);
      QTT_CUDA_TRY(cudaGetLastError());
    }
  }
  return QTT_OK;
}

qtt_status_t qtt_zipup_analyse(const char *subs, const qtt_trains_t *op, const qtt_trains_t *x, int32_t max_rank,
                               Shape &S) {
  return analyse(subs, op, x, max_rank, S);
}

}  // namespace qtt

using namespace qtt;

#if QTT_JAC_PROFILE
extern "C" int qtt_debug_jprof(unsigned long long *host, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host, qtt::g_jprof, sizeof(unsigned long long) * 24);
  if (reset) { unsigned long long z[24] = {}; cudaMemcpyToSymbol(qtt::g_jprof, z, sizeof(z)); }
  return 0;
}
#endif

extern "C" {

const char *qtt_last_error(void) { return qtt::g_err; }
const char *qtt_version(void) {
  return "libqtt 0.3 (sm_100a; fp64 zip-up: small- and large-member paths; fp32 variant with 3xTF32 tcgen05 contractions; complex128 and window-2 zip-ups)";
}

qtt_status_t qtt_zipup_capacity(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                int32_t max_rank, int32_t *cap) {
  Shape S;
  qtt_status_t st = analyse(subscripts, op, x, max_rank, S);
  if (st != QTT_OK) return st;
  if (!cap) { set_error("cap is NULL"); return QTT_EINVAL; }
  for (int q = 0; q <= S.L; ++q) cap[q] = S.cap[q];
  return QTT_OK;
}

size_t qtt_zipup_workspace_bytes(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                 const qtt_trains_t *out) {
  return qtt_zipup_workspace_bytes_flags(subscripts, op, x, out, 0);
}

size_t qtt_zipup_workspace_bytes_flags(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                       const qtt_trains_t *out, uint32_t flags) {
  const int dt = train_dtypes(op, x, out);
  if (dt < 0) { set_error("mixed dtypes: x, op and out must share one of QTT_F64, QTT_F32, QTT_C128"); return 0; }
  if (dt == 1) {                   // fp32 variant: fp64 staging of all three trains + the fp64 workspace
    F32Stage F;
    f32_stage(op, x, out, nullptr, F);
    const size_t inner =
        qtt_zipup_workspace_bytes_flags(subscripts, op ? &F.op64 : nullptr, &F.x64, out ? &F.out64 : nullptr, flags);
    return inner ? F.bytes + inner : 0;
  }
  // the output capacities the caller will pass bound the zip-up ranks (max_rank)
  int mr = 0;
  if (out && out->ranks && x)
    for (int q = 1; q < x->n_sites; ++q) mr = std::max(mr, (int)out->ranks[q]);
  Shape S;
  if (analyse(subscripts, op, x, mr, S) != QTT_OK) return 0;
  const int window = (flags & QTT_WINDOW2) ? 2 : 1;
  if (dt == 2 || window == 2) return member_workspace_bytes(S, dt == 2 ? 16 : 8, window);
  if (check_small_path(S) == QTT_OK) return layout(S).total;
  return large_workspace_bytes(S);
}

qtt_status_t qtt_zipup(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x, double eps,
                       int32_t max_rank, uint32_t flags, const qtt_trains_t *out, int32_t *out_ranks,
                       double *delta2, double *norm2, int32_t *status, const qtt_zipup_diag_t *diag,
                       void *workspace, size_t workspace_bytes, void *stream) {
  double *sigma = diag ? diag->sigma : nullptr;
  const int sigma_stride = diag ? diag->sigma_stride : 0;
  int *sweeps = diag ? diag->sweeps : nullptr;
  void *const *events = diag ? diag->events : nullptr;
  long long *cycles = diag ? (long long *)diag->phase_cycles : nullptr;
  g_err[0] = 0;
  if (!(eps >= 0.0 && eps < 1.0)) { set_error("eps %g outside [0,1)", eps); return QTT_EINVAL; }
  {
    const int dt = train_dtypes(op, x, out);
    if (dt < 0) { set_error("mixed dtypes: x, op and out must share one of QTT_F64, QTT_F32, QTT_C128"); return QTT_EINVAL; }
    if (dt == 1) {                 // fp32 variant (see qtt.h): widen, run with TF32 GEMMs, narrow
      if (!x || !out || !x->cores || !out->cores) { set_error("NULL train"); return QTT_EINVAL; }
      if (!workspace) { set_error("workspace is NULL"); return QTT_EINVAL; }
      F32Stage F;
      f32_stage(op, x, out, (char *)workspace, F);
      if (workspace_bytes < F.bytes) { set_error("workspace too small for the fp32 staging"); return QTT_ECAPACITY; }
      cudaStream_t s = (cudaStream_t)stream;
      qtt_status_t st = cvt_train(x, x->cores, F.xp.data(), true, s);
      if (st == QTT_OK && op) st = cvt_train(op, op->cores, F.op.data(), true, s);
      if (st != QTT_OK) return st;
      st = qtt_zipup(subscripts, op ? &F.op64 : nullptr, &F.x64, eps, max_rank, flags | kFlagTF32, &F.out64,
                     out_ranks, delta2, norm2, status, diag, (char *)workspace + F.bytes, workspace_bytes - F.bytes,
                     stream);
      if (st != QTT_OK) return st;
      return cvt_train(out, F.outp.data(), out->cores, false, s);
    }
  }
  Shape S;
  qtt_status_t st = analyse(subscripts, op, x, max_rank, S);
  if (st != QTT_OK) return st;
  if (!out || !out->cores || !out->ranks || !out_ranks || !delta2 || !norm2 || !status) {
    set_error("NULL output argument");
    return QTT_EINVAL;
  }
  if (out->n_sites != S.L || out->batch != S.B || out->n_legs != 1) {
    set_error("output train shape mismatch");
    return QTT_ESHAPE;
  }
  for (int q = 0; q <= S.L; ++q) {
    if (out->ranks[q] < S.cap[q]) {
      set_error("output capacity %d at bond %d below required %d", out->ranks[q], q, S.cap[q]);
      return QTT_ECAPACITY;
    }
  }
  for (int q = 0; q < S.L; ++q) {
    if (out->d_out[q] != S.d[q]) { set_error("output digit size mismatch at core %d", q); return QTT_ESHAPE; }
  }
  if (sigma && sigma_stride < 1) { set_error("sigma_stride < 1"); return QTT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  const bool cdt = train_dtypes(op, x, out) == 2;
  if (cdt || (flags & QTT_WINDOW2)) {      // complex128 (Fourier chain, f2) / window 2 (f4)
    g_err[0] = 0;
    if (events) QTT_CUDA_TRY(cudaEventRecord((cudaEvent_t)events[0], s));
    LargeIO io{out, out_ranks, delta2, norm2, sigma, sigma_stride, sweeps, status, eps, max_rank};
    qtt_status_t cst = member_zipup(S, op, x, flags, io, workspace, workspace_bytes, s, cycles, cdt,
                                    (flags & QTT_WINDOW2) ? 2 : 1, events);
    if (cst != QTT_OK) return cst;
    if (events) QTT_CUDA_TRY(cudaEventRecord((cudaEvent_t)events[3], s));
    return QTT_OK;
  }
  if (check_small_path(S) != QTT_OK) {
    // large-member path (site matrices with more than 128 rows): one member at a time
    g_err[0] = 0;
    QTT_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), s));
    if (events) QTT_CUDA_TRY(cudaEventRecord((cudaEvent_t)events[0], s));
    if (events) QTT_CUDA_TRY(cudaEventRecord((cudaEvent_t)events[1], s));
    if (events) QTT_CUDA_TRY(cudaEventRecord((cudaEvent_t)events[2], s));
    LargeIO io{out, out_ranks, delta2, norm2, sigma, sigma_stride, sweeps, status, eps, max_rank};
    qtt_status_t lst = large_zipup(S, op, x, flags, io, workspace, workspace_bytes, s);
    if (lst != QTT_OK) return lst;
    if (events) QTT_CUDA_TRY(cudaEventRecord((cudaEvent_t)events[3], s));
    return QTT_OK;
  }
  const WsLayout W = layout(S);
  if (workspace_bytes < W.total || !workspace) {
    set_error("workspace %zu bytes < required %zu", workspace_bytes, W.total);
    return QTT_ECAPACITY;
  }
  char *ws = (char *)workspace;
  double *Xo = (double *)(ws + W.xo), *Oo = (double *)(ws + W.oo), *G = (double *)(ws + W.g);
  double *T = (double *)(ws + W.t), *Xb = (double *)(ws + W.x);
  int *xr = (int *)(ws + W.xr), *orr = (int *)(ws + W.orr);

  // dynamic-smem opt-in on the current device, every call: the attribute is per device and the
  // call is cheap and thread-safe (qtt.h promises reentrant calls from any thread / device)
  QTT_CUDA_TRY(cudaFuncSetAttribute(k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSiteSmemBytes));
  QTT_CUDA_TRY(cudaFuncSetAttribute(k_orth, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(kOrthSmemDoubles * sizeof(double))));
  QTT_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), s));

  auto record = [&](int i) -> cudaError_t {
    return events ? cudaEventRecord((cudaEvent_t)events[i], s) : cudaSuccess;
  };
  QTT_CUDA_TRY(record(0));
  // a1: right-orthonormalise the operands
  {
    OrthArgs oa;
    memset(&oa, 0, sizeof(oa));
    oa.L = S.L; oa.orth = 1; oa.shared = 0;
    for (int q = 0; q < S.L; ++q) { oa.legs[q] = S.dj[q]; oa.src[q] = (const double *)x->cores[q]; oa.off[q] = S.xoff[q]; }
    for (int q = 0; q <= S.L; ++q) oa.r0[q] = S.xr[q];
    oa.dst = Xo; oa.dst_bs = S.xo_elems; oa.rk = xr;
    k_orth<<<S.B, kThreads, kOrthSmemDoubles * sizeof(double), s>>>(oa);
    QTT_CUDA_TRY(cudaGetLastError());
  }
  if (S.kind != TRUNCATE) {
    OrthArgs oa;
    memset(&oa, 0, sizeof(oa));
    oa.L = S.L; oa.orth = (flags & QTT_NO_OPERATOR_ORTH) ? 0 : 1; oa.shared = S.shared_op;
    for (int q = 0; q < S.L; ++q) {
      oa.legs[q] = (S.kind == MATVEC) ? S.d[q] * S.dj[q] : S.d[q];
      oa.src[q] = (const double *)op->cores[q];
      oa.off[q] = S.ooff[q];
    }
    for (int q = 0; q <= S.L; ++q) oa.r0[q] = S.orr[q];
    oa.dst = Oo; oa.dst_bs = S.oo_elems; oa.rk = orr;
    // a shared operator is orthonormalised once; its ranks are then broadcast per member
    const int nb = S.shared_op ? 1 : S.B;
    k_orth<<<nb, kThreads, kOrthSmemDoubles * sizeof(double), s>>>(oa);
    QTT_CUDA_TRY(cudaGetLastError());
    if (S.shared_op && S.B > 1) {
      k_bcast_row<<<(S.B * (S.L + 1) + 255) / 256, 256, 0, s>>>(orr, S.L + 1, S.B);
      QTT_CUDA_TRY(cudaGetLastError());
    }
  } else {
    QTT_CUDA_TRY(cudaMemsetAsync(orr, 0, sizeof(int) * (S.L + 1) * S.B, s));
  }

  QTT_CUDA_TRY(record(1));
  // a2..a7: the sweep over sites, one persistent launch for all members
  {
    SweepArgs a;
    memset(&a, 0, sizeof(a));
    a.L = S.L; a.B = S.B; a.kind = S.kind; a.shared_op = S.shared_op;
    for (int q = 0; q < S.L; ++q) {
      a.d[q] = S.d[q]; a.dj[q] = S.dj[q];
      a.xoff[q] = S.xoff[q]; a.ooff[q] = S.ooff[q];
      a.Cq[q] = (double *)out->cores[q];
      a.Cq_bs[q] = (long long)out->ranks[q] * S.d[q] * out->ranks[q + 1];
    }
    a.Xo = Xo; a.Xo_bs = S.xo_elems;
    a.Oo = (S.kind == TRUNCATE) ? nullptr : Oo;
    a.Oo_bs = S.oo_elems;
    a.xr = xr; a.orr = orr; a.yr = out_ranks;
    a.G = G; a.G_bs = S.g_elems; a.T = T; a.T_bs = S.t_elems; a.X = Xb; a.X_bs = S.x_elems;
    int *sched = (int *)(ws + W.sched);
    a.task_counter = sched; a.done = sched + 1;
    a.delta2 = delta2; a.norm2 = norm2; a.sigma = sigma; a.sigma_stride = sigma_stride; a.sweeps = sweeps;
    a.cycles = cycles; a.status = status; a.eps = eps; a.max_rank = max_rank;
    QTT_CUDA_TRY(cudaMemsetAsync(sched, 0, sizeof(int) * (1 + S.B), s));
    int dev = 0, sms = 0;
    QTT_CUDA_TRY(cudaGetDevice(&dev));
    QTT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // at most B tasks are runnable at once (a member's sites are sequential), and the per-CTA
    // T / X slots of the workspace number B
    const int grid = std::max(1, std::min(sms, S.B));
    QTT_CUDA_TRY(record(2));
    k_sweep<<<grid, kST, kSiteSmemBytes, s>>>(a);
    QTT_CUDA_TRY(cudaGetLastError());
    QTT_CUDA_TRY(record(3));
  }
  return QTT_OK;
}

}  // extern "C"
