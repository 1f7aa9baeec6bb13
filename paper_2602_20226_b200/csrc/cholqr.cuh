// cholqr.cuh -- a3 for the large-member path's wide site matrices (m <= n): the R of T^H by
// CholeskyQR2 on FP64 DMMA GEMMs, with the Householder QR (k_qr_coop) as the fallback.
//
//   W  = T T^T            (m x m Gram, split-K DMMA GEMM + fixed-order reduction)
//   R1 = chol(W)          (W = R1^T R1, blocked right-looking, cooperative)
//   Q1^T = R1^-T T        (explicit triangular inverse, then a DMMA GEMM; Q1^T in Tw)
//   W2 = Q1^T Q1          (Gram of the first pass's Q1, split-K)
//   R2 = chol(W2), R = R2 R1
//
// CholeskyQR2 is backward stable -- T^H = Q R + E with |E| = O(u)|T| and Q^T Q = I + O(u) --
// whenever the first pass's Q1 is well conditioned, i.e. |Q1^T Q1 - I| < 1 (Yamamoto,
// Nakatsukasa, Yanagisawa, Fukaya 2015).  The kernels check exactly that: both Cholesky
// factorisations must find positive pivots and |W2 - I|_F <= 1/2; otherwise the flag `ok`
// stays 0 and the Householder QR runs on the same site (rank-deficient or ill-conditioned T:
// cfg4's stencil products, the a o 1 known-answer input).  R then has the singular values of
// T to O(u)|T| absolute, the accuracy the one-sided Jacobi (a4) needs.  (SURVEY.md §8(a) a3
// rejects plain Gram / CholeskyQR for exactly the ill-conditioned case the gate routes away.)
#pragma once
#include "common.cuh"
#include "gemm.cuh"

namespace qtt {

constexpr int kCholNb = 32;                 // Cholesky / triangular-inverse block size

struct CholArgs {
  double *W;              // m x m row-major (ld m): in the Gram, out R (upper, zeros below)
  double *Dinv;           // [nblk][nb*nb] inverses of the diagonal blocks of R (row-major)
  const int *mdim;        // device: m (the site's rows)
  int *ok;                // in/out gate: cleared on a non-positive / non-finite pivot
  double *dev;            // |W - I|_F^2 of the input (second pass) or NULL
  double dev_max;         // gate: ok <- 0 when *dev > dev_max (second pass)
  GridBar *bar;
  int G;
};

// Cholesky of one 32 x 32 diagonal block in shared memory (upper: D = U^T U), then U^-1 into
// Ui (which has 32 spare doubles after the block) -- one warp: lane c holds column c in
// registers, row j (row r) of U reaches the other lanes through one shared-memory row per step
// (broadcast loads); 1/sqrt by the MUFU seed + Halley step and the inverse by multiplication
// with the kept reciprocals (measured 20k vs 60k cycles for the shared-memory loop version);
// the calling CTA's other warps skip it.  *fail set on a non-positive / non-finite pivot.
__device__ void chol_diag_block(double *D, double *Ui, int nb, int *fail) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    double *row = Ui + 32 * 32;
    double u[32], rpv[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) u[r] = D[r * 32 + lane];
    bool bad = false;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      row[lane] = u[j];                          // row j of the partially factored block
      __syncwarp();
      double d = row[j];
      if (!(d > 0.0) || !isfinite(d) || d < DBL_MIN) { bad = true; d = 1.0; }
      const double rp = fast_rsqrt(d), piv = d * rp;
      rpv[j] = rp;
      const double ujc = (lane > j) ? u[j] * rp : ((lane == j) ? piv : u[j]);
      u[j] = ujc;
#pragma unroll
      for (int r = j + 1; r < 32; ++r) {
        const double ujr = row[r] * rp;           // U[j][r]
        if (r <= lane) u[r] = fma(-ujr, ujc, u[r]);
      }
      __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r > lane) u[r] = 0.0;
    // X = U^-1, column `lane`: X[r][c] = (delta_rc - sum_{l>r} U[r][l] X[l][c]) / U[r][r]
    double x[32];
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      const int r = 31 - rr;
      row[lane] = u[r];                          // U[r][lane]
      __syncwarp();
      double s0 = (r == lane) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int l = r + 1; l < 32; ++l) {
        const double t = row[l] * x[l];
        if ((l & 3) == 0) s0 -= t; else if ((l & 3) == 1) s1 -= t; else if ((l & 3) == 2) s2 -= t; else s3 -= t;
      }
      x[r] = (r > lane) ? 0.0 : ((s0 + s1) + (s2 + s3)) * rpv[r];
      __syncwarp();
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) { D[r * 32 + lane] = u[r]; Ui[r * 32 + lane] = x[r]; }
    if (__any_sync(0xffffffffu, bad) && lane == 0) *fail = 1;
  }
  (void)nb;
  __syncthreads();
}

// Blocked right-looking Cholesky, W <- R (upper), one cooperative launch:
//   for each block row kb: CTA 0 factors the diagonal block (and its inverse); all CTAs form
//   the row panel R[kb][j] = U^-T W[kb][j]; all CTAs update the trailing upper blocks.
__global__ void __launch_bounds__(kThreads, 1) k_chol_coop(CholArgs a) {
  __shared__ double sA[kCholNb * kCholNb], sB[kCholNb * kCholNb + kCholNb], sC[kCholNb * kCholNb];
  __shared__ int s_fail;
  const int m = *a.mdim, nb = kCholNb, g = blockIdx.x, tid = threadIdx.x;
  if (m <= 0) return;
  if (*a.ok == 0) return;                          // uniform: an earlier step already failed
  if (a.dev && !(*a.dev <= a.dev_max)) {           // second pass: Q1 too far from orthonormal (or NaN)
    if (g == 0 && tid == 0) *a.ok = 0;
    return;
  }
  const int nblk = (m + nb - 1) / nb;
  auto ld = [&](double *dst, int br, int bc) {     // block (br, bc) of W into smem, zero padded
    for (int idx = tid; idx < nb * nb; idx += kThreads) {
      const int r = br * nb + idx / nb, c = bc * nb + idx % nb;
      dst[idx] = (r < m && c < m) ? a.W[(size_t)r * m + c] : ((r == c) ? 1.0 : 0.0);
    }
  };
  auto st = [&](const double *src, int br, int bc) {
    for (int idx = tid; idx < nb * nb; idx += kThreads) {
      const int r = br * nb + idx / nb, c = bc * nb + idx % nb;
      if (r < m && c < m) a.W[(size_t)r * m + c] = src[idx];
    }
  };
  auto factor_diag = [&](int kb, double *blk) {    // CTA 0: blk (smem) holds W[kb][kb]
    if (tid == 0) s_fail = 0;
    __syncthreads();
    chol_diag_block(blk, sB, nb, &s_fail);
    st(blk, kb, kb);
    for (int idx = tid; idx < nb * nb; idx += kThreads) a.Dinv[(size_t)kb * nb * nb + idx] = sB[idx];
    if (tid == 0 && s_fail) *a.ok = 0;
    __syncthreads();
  };
  if (g == 0) {
    ld(sA, 0, 0);
    factor_diag(0, sA);
  }
  for (int kb = 0; kb < nblk; ++kb) {
    grid_sync(a.bar, a.G, 21);                     // diagonal block kb factored (by CTA 0)
    if (__ldcg(a.ok) == 0) return;                 // uniform after the barrier
    // row panel: R[kb][j] = Dinv^T W[kb][j]  (j > kb)
    for (int jb = kb + 1 + g; jb < nblk; jb += a.G) {
      for (int idx = tid; idx < nb * nb; idx += kThreads) sA[idx] = __ldcg(a.Dinv + (size_t)kb * nb * nb + idx);
      ld(sB, kb, jb);
      __syncthreads();
      for (int idx = tid; idx < nb * nb; idx += kThreads) {
        const int r = idx / nb, c = idx % nb;
        double sacc = 0.0;
        for (int l = 0; l <= r; ++l) sacc = fma(sA[l * nb + r], sB[l * nb + c], sacc);   // (Dinv^T)[r][l] = Dinv[l][r]
        sC[idx] = sacc;
      }
      __syncthreads();
      st(sC, kb, jb);
      __syncthreads();
    }
    grid_sync(a.bar, a.G, 22);
    // trailing: W[ib][jb] -= R[kb][ib]^T R[kb][jb]  (kb < ib <= jb)
    // CTA 0 takes only tile (0, 0) -- the next diagonal block, which it then factors (the
    // critical path); the other tiles go to CTAs 1..G-1
    const int nt = nblk - kb - 1;
    const int t0 = (g == 0) ? 0 : g, tstep = (g == 0) ? (1 << 30) : max(a.G - 1, 1);
    for (int t = (a.G == 1) ? g : t0; t < nt * (nt + 1) / 2; t += (a.G == 1) ? 1 : tstep) {
      int ib = 0, rem = t;                          // t -> (ib <= jb) upper-triangular pair
      while (rem >= nt - ib) { rem -= nt - ib; ++ib; }
      const int jb = ib + rem;
      const int IB = kb + 1 + ib, JB = kb + 1 + jb;
      for (int idx = tid; idx < nb * nb; idx += kThreads) {
        const int r = kb * nb + idx / nb;
        const int c1 = IB * nb + idx % nb, c2 = JB * nb + idx % nb;
        sA[idx] = (r < m && c1 < m) ? __ldcg(a.W + (size_t)r * m + c1) : 0.0;
        sB[idx] = (r < m && c2 < m) ? __ldcg(a.W + (size_t)r * m + c2) : 0.0;
      }
      ld(sC, IB, JB);
      __syncthreads();
      for (int idx = tid; idx < nb * nb; idx += kThreads) {
        const int r = idx / nb, c = idx % nb;
        double sacc = sC[idx];
        for (int l = 0; l < nb; ++l) sacc = fma(-sA[l * nb + r], sB[l * nb + c], sacc);
        sC[idx] = sacc;
      }
      __syncthreads();
      if (t == 0) factor_diag(IB, sC);              // the next diagonal block, right after its update
      else st(sC, IB, JB);
      __syncthreads();
    }
  }
  // zeros below the diagonal (R is consumed as a full row-major matrix)
  for (long long idx = (long long)g * kThreads + tid; idx < (long long)m * m; idx += (long long)a.G * kThreads) {
    const int r = (int)(idx / m), c = (int)(idx % m);
    if (c < r) a.W[idx] = 0.0;
  }
}

// Rinv = R^-1 (upper, m x m row-major): one CTA per block column jb, back substitution over
// the block rows, X[jb][jb] = Dinv[jb], X[ib][jb] = -Dinv[ib] sum_{l=ib+1..jb} R[ib][l] X[l][jb]
struct TrinvArgs {
  const double *R, *Dinv;
  double *X;
  const int *mdim;
  const int *ok;
};
__global__ void __launch_bounds__(kThreads) k_trinv(TrinvArgs a) {
  __shared__ double sA[kCholNb * kCholNb], sB[kCholNb * kCholNb], sC[kCholNb * kCholNb];
  const int m = *a.mdim, nb = kCholNb, tid = threadIdx.x, jb = blockIdx.x;
  if (*a.ok == 0 || m <= 0) return;
  const int nblk = (m + nb - 1) / nb;
  if (jb >= nblk) return;
  auto stx = [&](const double *src, int br) {
    for (int idx = tid; idx < nb * nb; idx += kThreads) {
      const int r = br * nb + idx / nb, c = jb * nb + idx % nb;
      if (r < m && c < m) a.X[(size_t)r * m + c] = src[idx];
    }
  };
  for (int idx = tid; idx < nb * nb; idx += kThreads) sC[idx] = a.Dinv[(size_t)jb * nb * nb + idx];
  __syncthreads();
  stx(sC, jb);
  for (long long idx = tid; idx < (long long)(m - min(m, (jb + 1) * nb)) * nb; idx += kThreads) {   // zeros below
    const int r = (jb + 1) * nb + (int)(idx / nb), c = jb * nb + (int)(idx % nb);
    if (c < m) a.X[(size_t)r * m + c] = 0.0;
  }
  __syncthreads();
  for (int ib = jb - 1; ib >= 0; --ib) {
    // sC = sum_{l=ib+1..jb} R[ib][l] X[l][jb]
    for (int idx = tid; idx < nb * nb; idx += kThreads) sC[idx] = 0.0;
    __syncthreads();
    for (int lb = ib + 1; lb <= jb; ++lb) {
      for (int idx = tid; idx < nb * nb; idx += kThreads) {
        const int r = idx / nb, c = idx % nb;
        const int gr = ib * nb + r, gl = lb * nb + c;
        sA[idx] = (gr < m && gl < m) ? a.R[(size_t)gr * m + gl] : 0.0;
        const int xr = lb * nb + r, xc = jb * nb + c;
        sB[idx] = (xr < m && xc < m) ? a.X[(size_t)xr * m + xc] : 0.0;
      }
      __syncthreads();
      for (int idx = tid; idx < nb * nb; idx += kThreads) {
        const int r = idx / nb, c = idx % nb;
        double sacc = sC[idx];
        for (int l = 0; l < nb; ++l) sacc = fma(sA[r * nb + l], sB[l * nb + c], sacc);
        sC[idx] = sacc;
      }
      __syncthreads();
    }
    for (int idx = tid; idx < nb * nb; idx += kThreads) sA[idx] = a.Dinv[(size_t)ib * nb * nb + idx];
    __syncthreads();
    for (int idx = tid; idx < nb * nb; idx += kThreads) {
      const int r = idx / nb, c = idx % nb;
      double sacc = 0.0;
      for (int l = r; l < nb; ++l) sacc = fma(sA[r * nb + l], sC[l * nb + c], sacc);
      sB[idx] = -sacc;
    }
    __syncthreads();
    stx(sB, ib);
    __syncthreads();
  }
}

// fixed-order sum of split-K partials: W = sum_s P[s] (m x m, ld m); dev += |W - I|_F^2
struct RedArgs {
  const double *P;
  long long pstride;
  int S;
  const int *mdim;
  const int *ok;
  double *W;
  double *dev;
};
__global__ void k_gram_reduce(RedArgs a) {
  __shared__ double red[kThreads / 32];
  const int m = *a.mdim;
  if (*a.ok == 0) return;
  double dv = 0.0;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)m * m;
       idx += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(idx / m), c = (int)(idx % m);
    // the Gram GEMMs compute the upper tiles only (GemmSpec.upper): read (min, max)
    const long long src = (c >= r) ? idx : (long long)c * m + r;
    double sacc = 0.0;
    for (int s = 0; s < a.S; ++s) sacc += a.P[(size_t)s * a.pstride + src];
    a.W[idx] = sacc;
    const double e = sacc - ((r == c) ? 1.0 : 0.0);
    dv = fma(e, e, dv);
  }
  if (a.dev) {
    dv = block_sum(dv, red);
    if (threadIdx.x == 0) atomicAdd(a.dev, dv);
  }
}

}  // namespace qtt
