// large.cu -- large-member path of qtt_zipup: site matrices with m > 128 rows
// (BASELINE.json configs[1..3] at full size: T up to 512 x 65536 (cfg3) or 2560 x 1000 (cfg4)).
//
// One member at a time (these configs are single zip-ups); every kernel reads the site's
// dimensions from a device SiteDims record written by k_plan, so ranks stay on the device
// and grids are sized by capacity (surplus CTAs exit).  Per site q:
//   a2  k_gemm_dmma (strided batched FP64 DMMA GEMM, gemm.cuh) [+ k_mpo_apply]  T = contract(G, x_q, op_q)
//   a3  m <= n: k_qr_coop  -- cooperative, row-distributed Householder QR of T^H with grid
//                             barriers (16-column panels, WY trailing update, fixed-order
//                             reductions); robust to the exact rank deficiency that cfg2/cfg4
//                             site matrices show (kappa ~ 1e16), unlike Cholesky-QR.
//       m >  n: k_transpose -- A = T
//   a4  k_jacobi_coop -- one-sided Jacobi, block round-robin over CTAs, columns in shared
//                        memory, exact dot products, grid barrier per block round
//   a5/a6 k_finish (sigma, sort, truncation, emit U_k) + k_gemm_dmma carry G = U_k^T T
//   a7  k_last
// Operands too large for the shared-memory a1 kernel are right-orthonormalised by the
// mirrored truncate sweep (an SVD gauge instead of QR: the zip-up result is gauge
// invariant).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include <vector>

#include "large.cuh"
#include "gemm.cuh"
#include "gemm_tf32.cuh"

namespace qtt {

// ------------------------------------------------------------------ grid barrier

struct GridBar {
  unsigned count;
  unsigned gen;
  unsigned err;
  unsigned pad;
};

// All CTAs of a cooperative launch.  Release/acquire at gpu scope; the fence after the
// acquire also invalidates this SM's L1 so data written by other CTAs is re-read from L2.
// A barrier that does not complete within ~seconds records an error (reported through the
// zip-up status word) and lets the kernel finish instead of hanging the GPU.
__device__ __forceinline__ void grid_sync(GridBar *gb, unsigned nblocks, int tag = 0) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&gb->gen) : "memory");
    __threadfence();
    const unsigned arrived = atomicAdd(&gb->count, 1u);
    if (arrived == nblocks - 1) {
      atomicExch(&gb->count, 0u);
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&gb->gen), "r"(g + 1) : "memory");
    } else {
      unsigned v;
      long long spins = 0;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&gb->gen) : "memory");
        if (v == g) __nanosleep(32);
        if (++spins > (1LL << 24)) {
          if (atomicExch(&gb->err, 1u) == 0u)
            printf("qtt grid barrier timeout: tag %d cta %d/%u gen %u count %u\n", tag, (int)blockIdx.x, nblocks, g,
                   *((volatile unsigned *)&gb->count));
          break;
        }
      } while (v == g);
    }
    __threadfence();
  }
  __syncthreads();
}

// ------------------------------------------------------------------ site plan

struct SiteDims {
  int chi, r, r2, w, w2, d, dj, m, n, p, direct, k;
  int kcap;        // > 0: k <= kcap besides max_rank (the sharded zip-up's true column count)
};

struct PlanArgs {
  int q, L, kind, d, dj;
  const int *xr, *orr, *yr;     // member-offset rank rows
  const double *Xq, *Oq;
  double *G, *X, *T, *Cq;
  SiteDims *dims;
  GemmSpec *spec;               // [0] state GEMM, [1] Hadamard apply, [2] carry (k filled later)
};

__global__ void k_plan(PlanArgs a) {
  if (threadIdx.x != 0) return;
  SiteDims D;
  D.chi = (a.q == 0) ? 1 : a.yr[a.q];
  D.r = a.xr[a.q]; D.r2 = a.xr[a.q + 1];
  D.w = 1; D.w2 = 1;
  if (a.kind != TRUNCATE) { D.w = a.orr[a.q]; D.w2 = a.orr[a.q + 1]; }
  D.d = a.d; D.dj = a.dj;
  D.m = D.chi * D.d; D.n = D.w2 * D.r2;
  D.direct = (D.m > D.n);
  D.p = D.direct ? D.n : D.m;
  D.k = 0;
  D.kcap = 0;
  *a.dims = D;
  GemmSpec g0{};   // X = G (chi*w x r) * x_q (r x dj*r2)   [truncate: T = G (chi x r) * x_q]
  g0.M = D.chi * D.w; g0.K = D.r; g0.N = ((a.kind == HADAMARD || a.kind == TRUNCATE) ? D.d : D.dj) * D.r2;
  g0.nz1 = 1; g0.nz2 = 1;
  g0.A = a.G; g0.sam = g0.K; g0.sak = 1;
  g0.B = a.Xq; g0.sbk = g0.N; g0.sbn = 1;
  g0.C = (a.kind == TRUNCATE) ? a.T : a.X; g0.scm = g0.N; g0.scn = 1;
  a.spec[0] = g0;
  GemmSpec g1{};   // Hadamard: T[c,i,a2,b2] = sum_a A[a,i,a2] X[c,a,i,b2], batched over (c, i)
  g1.M = D.w2; g1.N = D.r2; g1.K = D.w; g1.nz1 = D.chi; g1.nz2 = D.d;
  g1.A = a.Oq; g1.sam = 1; g1.sak = (long long)D.d * D.w2; g1.sa1 = 0; g1.sa2 = D.w2;
  g1.B = a.X; g1.sbk = (long long)D.d * D.r2; g1.sbn = 1;
  g1.sb1 = (long long)D.w * D.d * D.r2; g1.sb2 = D.r2;
  g1.C = a.T; g1.scm = D.r2; g1.scn = 1; g1.sc1 = (long long)D.d * D.w2 * D.r2; g1.sc2 = (long long)D.w2 * D.r2;
  a.spec[1] = g1;
}

// DMMA GEMM (gemm.cuh) over capacity tiles; a_kcontig selects A's layout (row-major A,
// sak == 1, vs. transposed views with sam == 1).
static void launch_gemm_spec(const GemmSpec *spec, long long Mcap, long long Ncap, long long nz1cap, long long nz2cap,
                             bool a_kcontig, bool tf32, cudaStream_t s) {
  if (tf32) {        // fp32 variant: 3xTF32 on tcgen05 (gemm_tf32.cuh)
    const long long tm = (Mcap + tf32g::TM - 1) / tf32g::TM, tn = (Ncap + tf32g::TN - 1) / tf32g::TN;
    dim3 grid((unsigned)(tm * tn), 1, (unsigned)(nz1cap * nz2cap));
    if (a_kcontig)
      k_gemm_tf32<true><<<grid, 256, tf32g::SMEM_BYTES, s>>>(spec, (int)tn, (int)nz2cap);
    else
      k_gemm_tf32<false><<<grid, 256, tf32g::SMEM_BYTES, s>>>(spec, (int)tn, (int)nz2cap);
    return;
  }
  const long long tm = (Mcap + dgemm::TM - 1) / dgemm::TM, tn = (Ncap + dgemm::TN - 1) / dgemm::TN;
  dim3 grid((unsigned)(tm * tn), 1, (unsigned)(nz1cap * nz2cap));
  if (a_kcontig)
    k_gemm_dmma<true><<<grid, 256, dgemm::SMEM_BYTES, s>>>(spec, (int)tn, (int)nz2cap);
  else
    k_gemm_dmma<false><<<grid, 256, dgemm::SMEM_BYTES, s>>>(spec, (int)tn, (int)nz2cap);
}

// T[c,i,w2,r2] = sum_{w,j} X[c,w,j,r2] W[w,i,j,w2]
__global__ void k_mpo_apply(const SiteDims *dims, const double *X, const double *W, double *T) {
  const SiteDims D = *dims;
  const long long total = (long long)D.m * D.n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int rr2 = (int)(idx % D.r2);
    long long t1 = idx / D.r2;
    const int ww2 = (int)(t1 % D.w2); t1 /= D.w2;
    const int ii = (int)(t1 % D.d);
    const long long c = t1 / D.d;
    double s = 0.0;
    for (int ww = 0; ww < D.w; ++ww)
      for (int jj = 0; jj < D.dj; ++jj)
        s = fma(X[((c * D.w + ww) * D.dj + jj) * D.r2 + rr2], W[(((long long)ww * D.d + ii) * D.dj + jj) * D.w2 + ww2], s);
    T[idx] = s;
  }
}

__global__ void k_copy_T(const SiteDims *dims, const double *T, double *Tw, double *A, const int *skip = nullptr,
                         const int *skip_tall = nullptr) {
  const SiteDims D = *dims;
  if (!D.direct && skip && *skip) return;        // CholeskyQR2 produced R: the Householder copy is not needed
  if (D.direct && skip_tall && *skip_tall) return;   // tall CholeskyQR2 orthonormalised the site: no Jacobi
  const long long total = (long long)D.m * D.n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const double v = T[idx];
    if (D.direct) {   // A (m x n) column-major: A[j*m + row] = T[row*n + j]
      const long long row = idx / D.n, j = idx % D.n;
      A[j * D.m + row] = v;
    } else {
      Tw[idx] = v;
    }
  }
}

// ------------------------------------------------------------------ a3: CholeskyQR2 (cholqr.cuh)
}  // namespace qtt
#include "cholqr.cuh"
namespace qtt {

struct CqPlanArgs {
  const SiteDims *dims;
  int S, mmin;
  const double *T;
  double *Tw, *P, *Rinv, *R1, *R2, *Rout;
  long long pstride;
  GemmSpec *spec;          // [4]
  int *ok, *mdim;
  double *dev;
};

// decides whether the site takes CholeskyQR2 (wide: m <= n, m >= mmin) and fills its GEMM specs
__global__ void k_cq_plan(CqPlanArgs a) {
  if (threadIdx.x != 0) return;
  const SiteDims D = *a.dims;
  const int m = D.m, n = D.n;
  const int use = (!D.direct && m >= a.mmin && m <= n) ? 1 : 0;
  *a.ok = use;
  *a.mdim = use ? m : 0;
  *a.dev = 0.0;
  const int kc = ((n + a.S - 1) / a.S + 15) / 16 * 16;
  GemmSpec g{};
  // [0] P_s = T[:, chunk s] T[:, chunk s]^T   (A = T K-contiguous, B = T^T K-contiguous)
  g.M = use ? m : 0; g.N = m; g.K = n; g.nz1 = a.S; g.nz2 = 1; g.kchunk = kc;
  g.A = a.T; g.sam = n; g.sak = 1; g.sa1 = kc;
  g.B = a.T; g.sbk = 1; g.sbn = n; g.sb1 = kc;
  g.C = a.P; g.scm = m; g.scn = 1; g.sc1 = a.pstride;
  g.upper = 1;
  a.spec[0] = g;
  // [1] Q1^T = Rinv^T T (m x n): A[i][k] = Rinv[k][i] (M-contiguous, lower triangular), B = T
  GemmSpec h{};
  h.M = use ? m : 0; h.N = n; h.K = m; h.nz1 = 1; h.nz2 = 1; h.tri = 1;
  h.A = a.Rinv; h.sam = 1; h.sak = m;
  h.B = a.T; h.sbk = n; h.sbn = 1;
  h.C = a.Tw; h.scm = n; h.scn = 1;
  a.spec[1] = h;
  // [2] P_s = Q1^T Q1 partials
  GemmSpec g2 = g;
  g2.A = a.Tw; g2.B = a.Tw;
  a.spec[2] = g2;
  // [3] R = R2 R1 (row-major, ld m) -> Rout
  GemmSpec r{};
  r.M = use ? m : 0; r.N = m; r.K = m; r.nz1 = 1; r.nz2 = 1; r.tri = 2;
  r.A = a.R2; r.sam = m; r.sak = 1;
  r.B = a.R1; r.sbk = m; r.sbn = 1;
  r.C = a.Rout; r.scm = m; r.scn = 1;
  a.spec[3] = r;
}

// Tall variant for the exact orthonormalisation sweeps (a1: truncate with eps = 0, the site
// matrix T with m > n): T = Q R by CholeskyQR2 with Q explicit; the output core is Q (m x n,
// the SVD path's U_p up to an orthogonal n x n gauge -- a1's result is gauge-invariant, c-A3) and
// the carry is R, so no Jacobi runs.  Specs: [0] P_s = T^T T partials, [1] Q1 = T Rinv1 -> Tw,
// [2] P_s = Q1^T Q1 partials, [3] Q = Q1 Rinv2 -> C_q, [4] R = R2 R1 -> G.
struct CqtPlanArgs {
  const SiteDims *dims;
  int S, nmin;
  const double *T;
  double *Tw, *P, *Rinv, *R1, *R2, *Cq, *Gout;
  long long pstride;
  GemmSpec *spec;          // [5]
  int *ok, *ndim;
  double *dev;
};
__global__ void k_cqt_plan(CqtPlanArgs a) {
  if (threadIdx.x != 0) return;
  const SiteDims D = *a.dims;
  const int m = D.m, n = D.n;
  const int use = (D.direct && n >= a.nmin && m > n) ? 1 : 0;
  *a.ok = use;
  *a.ndim = use ? n : 0;
  *a.dev = 0.0;
  const int kc = ((m + a.S - 1) / a.S + 15) / 16 * 16;
  GemmSpec g{};            // [0] T^T T: A[i][k] = T[k][i] (M-contiguous), B = T
  g.M = use ? n : 0; g.N = n; g.K = m; g.nz1 = a.S; g.nz2 = 1; g.kchunk = kc;
  g.A = a.T; g.sam = 1; g.sak = n; g.sa1 = (long long)kc * n;
  g.B = a.T; g.sbk = n; g.sbn = 1; g.sb1 = (long long)kc * n;
  g.C = a.P; g.scm = n; g.scn = 1; g.sc1 = a.pstride;
  g.upper = 1;
  a.spec[0] = g;
  GemmSpec h{};            // [1] Q1 = T Rinv (m x n), Rinv upper triangular
  h.M = use ? m : 0; h.N = n; h.K = n; h.nz1 = 1; h.nz2 = 1; h.tri = 2;
  h.A = a.T; h.sam = n; h.sak = 1;
  h.B = a.Rinv; h.sbk = n; h.sbn = 1;
  h.C = a.Tw; h.scm = n; h.scn = 1;
  a.spec[1] = h;
  GemmSpec g2 = g;         // [2] Q1^T Q1
  g2.A = a.Tw; g2.B = a.Tw;
  a.spec[2] = g2;
  GemmSpec q = h;          // [3] Q = Q1 Rinv2 -> the output core
  q.A = a.Tw; q.C = a.Cq;
  a.spec[3] = q;
  GemmSpec r{};            // [4] R = R2 R1 -> the carry (n x n)
  r.M = use ? n : 0; r.N = n; r.K = n; r.nz1 = 1; r.nz2 = 1; r.tri = 2;
  r.A = a.R2; r.sam = n; r.sak = 1;
  r.B = a.R1; r.sbk = n; r.sbn = 1;
  r.C = a.Gout; r.scm = n; r.scn = 1;
  a.spec[4] = r;
}

// the tall site's a5/a6 bookkeeping when CholeskyQR2 was accepted: rank n, nothing discarded,
// the carry already in G (the sweep's own carry GEMM becomes empty)
__global__ void k_cqt_finish(const int *ok, SiteDims *dims, int *yr_next, double *delta2, GemmSpec *carry,
                             int *sweeps) {
  if (threadIdx.x != 0 || *ok == 0) return;
  const int n = dims->n;
  dims->k = n;
  *yr_next = n;
  *delta2 = 0.0;
  carry->M = 0;
  if (sweeps) *sweeps = 0;
}

// after a Cholesky: when the gate closed, the remaining CholeskyQR2 GEMMs become empty
__global__ void k_cq_gate(const int *ok, GemmSpec *spec, int from, int count = 4) {
  if (threadIdx.x != 0) return;
  if (*ok == 0)
    for (int i = from; i < count; ++i) spec[i].M = 0;
}

// ------------------------------------------------------------------ a3: cooperative QR

#ifndef QTT_QR_NB
#define QTT_QR_NB 16
#endif
constexpr int kNb = QTT_QR_NB;       // panel width (32 measured: cfg3 equal, cfg2 +10% -- the
                                     // column-step grid barriers, not the trailing passes, bound it)
constexpr int kQrRowsMax = 512;      // max T^H rows per CTA held in shared memory (panel)

struct QrArgs {
  const SiteDims *dims;
  double *Tw;          // m x n row-major; T^H column c = row c (length n)
  double *Rout;        // m x m row-major R (zeros below the diagonal) == A column-major
  double *part;        // [G][kNb * mcap]  partial sums
  double *wtot;        // [kNb * mcap]     reduced W
  double *gram;        // [kNb * kNb]      reduced Y^T Y
  double *bc;          // broadcast row-j values of the panel columns [2][32] (column parity)
  GridBar *bar;
  int G, RB, mcap;
  const int *skip;     // non-NULL and set: R already computed (CholeskyQR2 accepted): return
  double *tau_out;     // non-NULL: the Householder scalars tau_j are kept (explicit Q later)
};

// Reduce a per-CTA scalar triple of arrays: block sum of v over kThreads.
__device__ __forceinline__ double block_sum_l(double v, double *red) { return block_sum(v, red); }

__global__ void __launch_bounds__(kThreads, 1) k_qr_coop(QrArgs a) {
  extern __shared__ double smq[];
  const SiteDims D = *a.dims;
  if (D.direct) return;                         // uniform across the grid
  if (a.skip && *a.skip) return;
  const int m = D.m, n = D.n, g = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = g * a.RB, r1 = min(n, r0 + a.RB), nr = max(0, r1 - r0);
  double *P = smq;                              // [kNb][RB] panel (my rows)
  double *Y = P;                                // the same storage holds the reflectors (unit
                                                // diagonal explicit) once the panel is written back
  double *red = P + kNb * a.RB;                 // [kThreads/32]
  double *tw = red + 32;                        // [kNb*kNb] T_wy ; [kNb] tau ; [kNb] dots
  double *tau = tw + kNb * kNb;
  double *dots = tau + kNb;
  double *Mt = dots + kNb;                      // [kNb * 64] chunk of T_wy^T W
  const unsigned G = a.G;
  for (int j0 = 0; j0 < m; j0 += kNb) {
    const int nb = min(kNb, m - j0);
    // load the panel (T^H columns j0..j0+nb, my rows)
    for (int idx = tid; idx < nb * nr; idx += kThreads) {
      const int cc = idx / nr, i = idx % nr;
      P[cc * a.RB + i] = a.Tw[(size_t)(j0 + cc) * n + r0 + i];
    }
    __syncthreads();
    // Column steps with ONE grid barrier each: every CTA reduces, over its rows r > j, the
    // products x_j . x_cc for cc >= jj (cc == jj: the squared norm below the diagonal); the
    // owner of row j publishes x_cc[j].  Then v_j . x_cc = x_cc[j] + scale * sum_{r>j} x_j x_cc
    // (v_j = [1; scale x_j(r > j)]) needs no second reduction.  part / bc are double-buffered
    // by column parity (a slot is rewritten two barriers later, after every CTA read it).
    for (int jj = 0; jj < nb; ++jj) {
      const int j = j0 + jj, slot = (j & 1) * 32;
      for (int cc = jj + warp; cc < nb; cc += kWarps) {
        double d = 0.0;
        for (int i = lane; i < nr; i += 32)
          if (r0 + i > j) d = fma(P[jj * a.RB + i], P[cc * a.RB + i], d);
        d = warp_sum(d);
        if (lane == 0) {
          a.part[(size_t)g * kNb * a.mcap + slot + cc] = d;
          if (j >= r0 && j < r1) a.bc[slot + cc] = P[cc * a.RB + (j - r0)];
        }
      }
      grid_sync(a.bar, G, 1);
      double tj, beta, scale;
      {
        double s = 0.0;
        for (unsigned gg = 0; gg < G; ++gg) s += __ldcg(a.part + (size_t)gg * kNb * a.mcap + slot + jj);
        householder(__ldcg(a.bc + slot + jj), s, tj, beta, scale);
      }
      if (tid == 0) tau[jj] = tj;
      if (a.tau_out && g == 0 && tid == 0) a.tau_out[j] = tj;
      if (tid < kNb) {
        double w = 0.0;
        if (tid > jj && tid < nb && tj != 0.0) {
          double sd = 0.0;
          for (unsigned gg = 0; gg < G; ++gg) sd += __ldcg(a.part + (size_t)gg * kNb * a.mcap + slot + tid);
          w = tj * fma(scale, sd, __ldcg(a.bc + slot + tid));
        }
        dots[tid] = w;
      }
      __syncthreads();
      // per row (one thread owns a row of the panel): trailing panel columns -= w_cc v, then
      // v: rows > j scaled; row j -> beta (R diagonal), v_j = 1 implicit
      for (int i = tid; i < nr; i += kThreads) {
        const int r = r0 + i;
        const double x = P[jj * a.RB + i];
        if (r > j) {
          const double v = x * scale;
          for (int cc = jj + 1; cc < nb; ++cc) P[cc * a.RB + i] = fma(-dots[cc], v, P[cc * a.RB + i]);
          P[jj * a.RB + i] = v;
        } else if (r == j) {
          for (int cc = jj + 1; cc < nb; ++cc) P[cc * a.RB + i] -= dots[cc];
          P[jj * a.RB + i] = beta;
        }
      }
      __syncthreads();
    }
    // write the factored panel back (R entries and reflectors), build Y
    for (int idx = tid; idx < nb * nr; idx += kThreads) {
      const int cc = idx / nr, i = idx % nr, r = r0 + i, j = j0 + cc;
      const double pv = P[cc * a.RB + i];
      a.Tw[(size_t)j * n + r] = pv;
      Y[cc * a.RB + i] = (r > j) ? pv : (r == j ? 1.0 : 0.0);
    }
    for (int idx = tid; idx < kNb * a.RB; idx += kThreads)
      if (idx / a.RB >= nb) Y[idx] = 0.0;
    __syncthreads();
    const int c0 = j0 + nb;                     // trailing T^H columns c0..m-1
    if (c0 < m) {
      // partial W[k][c] = sum_r Y[r][k] C[r][c] (my rows) and partial Y^T Y
      for (int c = c0 + warp; c < m; c += kWarps) {
        double acc[kNb];
#pragma unroll
        for (int kk = 0; kk < kNb; ++kk) acc[kk] = 0.0;
        for (int i = lane; i < nr; i += 32) {
          const double x = a.Tw[(size_t)c * n + r0 + i];
#pragma unroll
          for (int kk = 0; kk < kNb; ++kk) acc[kk] = fma(Y[kk * a.RB + i], x, acc[kk]);
        }
#pragma unroll
        for (int kk = 0; kk < kNb; ++kk) {
          const double t = warp_sum(acc[kk]);
          if (lane == 0) a.part[(size_t)g * kNb * a.mcap + (size_t)kk * a.mcap + c] = t;
        }
      }
      double *gpart = a.part + (size_t)G * kNb * a.mcap;    // [G][kNb*kNb]
      for (int e = warp; e < kNb * kNb; e += kWarps) {
        const int k1 = e / kNb, k2 = e % kNb;
        double s = 0.0;
        for (int i = lane; i < nr; i += 32) s = fma(Y[k1 * a.RB + i], Y[k2 * a.RB + i], s);
        s = warp_sum(s);
        if (lane == 0) gpart[(size_t)g * kNb * kNb + e] = s;
      }
      grid_sync(a.bar, G, 3);
      // distributed reduction: CTA g sums columns c = c0 + g, c0 + g + G, ...
      for (int idx = tid; idx < kNb * ((m - c0 + (int)G - 1 - g) / (int)G); idx += kThreads) {
        const int kk = idx % kNb, t = idx / kNb, c = c0 + g + t * (int)G;
        if (c >= m) continue;
        double s = 0.0;
        for (unsigned gg = 0; gg < G; ++gg) s += a.part[(size_t)gg * kNb * a.mcap + (size_t)kk * a.mcap + c];
        a.wtot[(size_t)kk * a.mcap + c] = s;
      }
      if (g == 0)
        for (int e = tid; e < kNb * kNb; e += kThreads) {
          double s = 0.0;
          for (unsigned gg = 0; gg < G; ++gg) s += gpart[(size_t)gg * kNb * kNb + e];
          a.gram[e] = s;
        }
      grid_sync(a.bar, G, 4);
      // T_wy (upper triangular): T_jj = tau_j, T[0:j, j] = -tau_j * T[0:j,0:j] * (Y^T y_j)[0:j]
      if (tid == 0) {
        for (int e = 0; e < kNb * kNb; ++e) tw[e] = 0.0;
        for (int j = 0; j < nb; ++j) {
          tw[j * kNb + j] = tau[j];
          for (int i = 0; i < j; ++i) {
            double s = 0.0;
            for (int l = i; l < j; ++l) s += tw[i * kNb + l] * a.gram[l * kNb + j];
            tw[i * kNb + j] = -tau[j] * s;
          }
        }
      }
      __syncthreads();
      // C -= Y (T^T W): process trailing columns in chunks of 64
      for (int cb = c0; cb < m; cb += 64) {
        const int ncb = min(64, m - cb);
        for (int idx = tid; idx < kNb * ncb; idx += kThreads) {   // Mt[k][c] = sum_l T[l][k] W[l][c]
          const int kk = idx / ncb, c = idx % ncb;
          double s = 0.0;
          for (int l = 0; l <= kk; ++l) s = fma(tw[l * kNb + kk], a.wtot[(size_t)l * a.mcap + cb + c], s);
          Mt[kk * 64 + c] = s;
        }
        __syncthreads();
        for (int c = warp; c < ncb; c += kWarps) {
          double *col = a.Tw + (size_t)(cb + c) * n + r0;
          for (int i = lane; i < nr; i += 32) {
            double s = col[i];
#pragma unroll
            for (int kk = 0; kk < kNb; ++kk) s = fma(-Y[kk * a.RB + i], Mt[kk * 64 + c], s);
            col[i] = s;
          }
        }
        __syncthreads();
      }
    }
    grid_sync(a.bar, G, 5);
  }
  // R (m x m, row-major, lower part zero) from rows 0..m-1 of the factored T^H
  for (long long idx = (long long)g * kThreads + tid; idx < (long long)m * m; idx += (long long)G * kThreads) {
    const int j = (int)(idx / m), c = (int)(idx % m);
    a.Rout[idx] = (c >= j) ? a.Tw[(size_t)c * n + j] : 0.0;
  }
}

// ------------------------------------------------------------------ tall sites: QR first
// A direct site (m > n: T is taller than wide) whose Jacobi would run on m-row columns is first
// reduced by a Householder QR, T = Q R (k_qr_coop on T^T, the reflectors kept): the Jacobi then
// runs on the n x n columns of R (fewer rows per rotation, and a wider block), and its left
// singular vectors U_R become U_T = Q [U_R; 0] by applying the reflectors (k_qapply_coop).  The
// host marks a site a candidate when its capacities satisfy m_cap >= 2 n_cap, n_cap >= 32 (cfg4's
// d = 5 sites: 2560 x 1000, 1875 x 200); the device takes the route when the site is direct.  On a
// candidate the Jacobi's columns have at most n_cap rows either way, which sizes its block.

struct TqPlanArgs {
  const SiteDims *dims;   // the site
  SiteDims *dims_j;       // out: the Jacobi / finish dims (R's n x n, or a copy of the site's)
  SiteDims *dims_t;       // out: the QR's dims (T^T as a wide "T")
  SiteDims *dims_2;       // out: the second QR's dims (R1^T, n x n)
  int *tq, *ntq;          // out: 1 / 0 when the site takes the QR-first route
  const int *busy;        // non-NULL and set: the site is handled otherwise (tall CholeskyQR2)
};
__global__ void k_tq_plan(TqPlanArgs a) {
  if (threadIdx.x != 0) return;
  const SiteDims D = *a.dims;
  const int use = (D.direct && !(a.busy && *a.busy)) ? 1 : 0;
  *a.tq = use; *a.ntq = 1 - use;
  SiteDims J = D;
  if (use) { J.m = D.n; J.n = D.n; J.p = D.n; J.direct = 0; }
  J.k = 0;
  *a.dims_j = J;
  SiteDims T = D;
  T.m = D.n; T.n = D.m; T.p = D.n; T.direct = 0;
  *a.dims_t = T;
  T.n = D.n;
  *a.dims_2 = T;
}
// ||T||_F^2 partial sums (one per CTA): the QR runs on T scaled by a power of two with
// ||T||_F^2 in [1, 4) (as k_jacobi_coop does), so that no sum of squares in the Householder
// steps underflows for any input magnitude; R is scaled back exactly in k_tq_toA
__global__ void k_tq_sq(const SiteDims *dims, const int *tq, const double *T, double *part) {
  __shared__ double red[kWarps];
  if (!*tq) return;
  const long long mn = (long long)dims->m * dims->n;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < mn; i += (long long)gridDim.x * blockDim.x) {
    const double v = T[i];
    s = fma(v, v, s);
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
// Tw (n x m row-major) = 2^e T^T, so that k_qr_coop's "T^H" is the tall T (scaled)
__global__ void k_tq_copy(const SiteDims *dims, const int *tq, const double *T, const double *part, int nparts,
                          double *Tw, double *scale_out) {
  __shared__ double sc;
  if (!*tq) return;
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int t = 0; t < nparts; ++t) tot += part[t];
    double f = 1.0;
    if (tot > 0.0 && isfinite(tot)) f = ldexp(1.0, -(ilogb(tot) >> 1));
    sc = f;
    if (blockIdx.x == 0) *scale_out = f;
  }
  __syncthreads();
  const double f = sc;
  const SiteDims D = *dims;
  const long long mn = (long long)D.m * D.n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < mn; i += (long long)gridDim.x * blockDim.x) {
    const long long j = i / D.m, r = i % D.m;
    Tw[i] = T[r * D.n + j] * f;
  }
}
// A (n x n column-major) = R / 2^e: A[j*n + i] = R[i][j] (R row-major, upper); with `as_is`
// A = R's storage / 2^e (the column-major R^T; R may alias A)
__global__ void k_tq_toA(const SiteDims *dims, const int *tq, const double *R, const double *scale, double *A,
                         int as_is) {
  if (!*tq) return;
  const int n = dims->n;
  const double inv = 1.0 / *scale;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)n * n; i += (long long)gridDim.x * blockDim.x) {
    if (as_is) { A[i] = R[i] * inv; continue; }
    const int j = (int)(i / n), r = (int)(i % n);
    A[i] = (r <= j) ? R[(size_t)r * n + j] * inv : 0.0;
  }
}

struct QapplyArgs {
  const SiteDims *dims;   // the site (m rows, n reflectors)
  const SiteDims *dims_j; // k of the split
  const int *tq;
  const double *Yw;       // reflectors: column j in Yw[j*m + r], r > j (unit at r == j)
  const double *tau;      // [n]
  double *C;              // m x k row-major: in [U_R; garbage below n], out Q [U_R; 0]
  double *part, *wtot, *gram;
  GemmSpec *carry;        // the carry spec: K <- m
  GridBar *bar;
  int G, RB;
};
__global__ void __launch_bounds__(kThreads, 1) k_qapply_coop(QapplyArgs a) {
  extern __shared__ double smq[];
  if (!*a.tq) return;                          // uniform
  const SiteDims D = *a.dims;
  const int m = D.m, n = D.n, k = a.dims_j->k, g = blockIdx.x, tid = threadIdx.x, lane = tid & 31,
            warp = tid >> 5;
  const int r0 = g * a.RB, r1 = min(m, r0 + a.RB), nr = max(0, r1 - r0);
  double *Y = smq;                             // [kNb][RB]
  double *tw = Y + kNb * a.RB;                 // [kNb * kNb]
  double *Mt = tw + kNb * kNb;                 // [kNb * 64]
  const unsigned G = a.G;
  // rows >= n of C start at zero (C = [U_R; 0])
  for (long long idx = (long long)g * kThreads + tid; idx < (long long)(m - n) * k; idx += (long long)G * kThreads)
    a.C[(size_t)n * k + idx] = 0.0;
  grid_sync(a.bar, G, 31);
  const int npan = (n + kNb - 1) / kNb;
  for (int pan = npan - 1; pan >= 0; --pan) {
    const int j0 = pan * kNb, nb = min(kNb, n - j0);
    for (int idx = tid; idx < kNb * nr; idx += kThreads) {
      const int cc = idx / nr, i = idx % nr, r = r0 + i, j = j0 + cc;
      Y[cc * a.RB + i] = (cc >= nb) ? 0.0 : (r > j ? a.Yw[(size_t)j * m + r] : (r == j ? 1.0 : 0.0));
    }
    __syncthreads();
    // partial W[cc][c] = sum_r Y[r][cc] C[r][c] and partial Y^T Y over my rows
    for (int c = warp; c < k; c += kWarps) {
      double acc[kNb];
#pragma unroll
      for (int cc = 0; cc < kNb; ++cc) acc[cc] = 0.0;
      for (int i = lane; i < nr; i += 32) {
        const double x = a.C[(size_t)(r0 + i) * k + c];
#pragma unroll
        for (int cc = 0; cc < kNb; ++cc) acc[cc] = fma(Y[cc * a.RB + i], x, acc[cc]);
      }
#pragma unroll
      for (int cc = 0; cc < kNb; ++cc) {
        const double t = warp_sum(acc[cc]);
        if (lane == 0) a.part[((size_t)g * kNb + cc) * k + c] = t;
      }
    }
    double *gpart = a.part + (size_t)G * kNb * k;
    for (int e = warp; e < kNb * kNb; e += kWarps) {
      const int k1 = e / kNb, k2 = e % kNb;
      double sacc = 0.0;
      for (int i = lane; i < nr; i += 32) sacc = fma(Y[k1 * a.RB + i], Y[k2 * a.RB + i], sacc);
      sacc = warp_sum(sacc);
      if (lane == 0) gpart[(size_t)g * kNb * kNb + e] = sacc;
    }
    grid_sync(a.bar, G, 32);
    for (int idx = g * kThreads + tid; idx < kNb * k; idx += G * kThreads) {
      double sacc = 0.0;
      for (unsigned gg = 0; gg < G; ++gg) sacc += __ldcg(a.part + (size_t)gg * kNb * k + idx);
      a.wtot[idx] = sacc;
    }
    if (g == 0)
      for (int e = tid; e < kNb * kNb; e += kThreads) {
        double sacc = 0.0;
        for (unsigned gg = 0; gg < G; ++gg) sacc += __ldcg(gpart + (size_t)gg * kNb * kNb + e);
        a.gram[e] = sacc;
      }
    grid_sync(a.bar, G, 33);
    // T_wy of H_{j0} ... H_{j0+nb-1} (upper): T_jj = tau_j, T[0:j, j] = -tau_j T[0:j,0:j] (Y^T y_j)[0:j]
    if (tid == 0) {
      for (int e = 0; e < kNb * kNb; ++e) tw[e] = 0.0;
      for (int j = 0; j < nb; ++j) {
        const double tj = __ldcg(a.tau + j0 + j);
        tw[j * kNb + j] = tj;
        for (int i = 0; i < j; ++i) {
          double sacc = 0.0;
          for (int l = i; l < j; ++l) sacc += tw[i * kNb + l] * __ldcg(a.gram + l * kNb + j);
          tw[i * kNb + j] = -tj * sacc;
        }
      }
    }
    __syncthreads();
    // C -= Y (T W), columns in chunks of 64
    for (int cb = 0; cb < k; cb += 64) {
      const int ncb = min(64, k - cb);
      for (int idx = tid; idx < kNb * ncb; idx += kThreads) {
        const int kk = idx / ncb, c = idx % ncb;
        double sacc = 0.0;
        for (int l = kk; l < kNb; ++l) sacc = fma(tw[kk * kNb + l], __ldcg(a.wtot + (size_t)l * k + cb + c), sacc);
        Mt[kk * 64 + c] = sacc;
      }
      __syncthreads();
      for (int idx = tid; idx < nr * ncb; idx += kThreads) {
        const int i = idx / ncb, c = idx % ncb;
        double *cp = a.C + (size_t)(r0 + i) * k + cb + c;
        double sacc = *cp;
#pragma unroll
        for (int kk = 0; kk < kNb; ++kk) sacc = fma(-Y[kk * a.RB + i], Mt[kk * 64 + c], sacc);
        *cp = sacc;
      }
      __syncthreads();
    }
    grid_sync(a.bar, G, 34);
  }
  if (g == 0 && tid == 0) a.carry->K = m;        // the carry G = U_T^T T runs over the site's m rows
}

// ------------------------------------------------------------------ a4: cooperative Jacobi

struct JacArgs {
  const SiteDims *dims;
  double *A;               // m x p column-major, ld m
  GridBar *bar;
  int *flags;              // [3] rotating 'rotated in sweep s' flags
  int *ver;                // [NB] block versions: block b holds the result of global round ver[b]-1
  double *part;            // [G] per-CTA partial sums of ||A||_F^2
  double *nrm;             // [p] carried squared column norms between block rounds
  int noise_ok;            // eps > 1e-14: noise-level columns are truncated anyway (rot_pair)
  int G, WB;               // CTAs, block width (columns)
  int *sweeps_out;
  int *status;
  const int *skip;         // non-NULL and set: the site was orthonormalised by CholeskyQR2 (a1 sweeps)
};

// One Jacobi pair (one warp): exact dot product, column norms nrm_i / nrm_j carried in shared
// memory by the rotation identities (exact refresh on cancellation, LAPACK dgesvj practice),
// division-free MUFU-seeded angle (same formulas as the small path, jacobi.cuh).  Pairs with
// a column at rounding-noise level (|a|^2 <= noise = eps^2 ||A||_F^2) are left alone: their
// relative orthogonality is below what fp64 can resolve, rotating them moves O(eps ||A||)
// mass, and they would otherwise keep the sweeps going (cfg4's rank-deficient sites).  Only
// when the truncation eps > 1e-14 guarantees such columns are discarded (eps = 0 -- the
// exact a1 sweeps -- keeps them, and then they must come out orthonormal).
__device__ __forceinline__ double col_norm2(const double *c, int m) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int r = lane; r < m; r += 32) s = fma(c[r], c[r], s);
  return warp_sum(s);
}

// Rotation of one pair given (al, be, ga); shared by the scalar and the paired-row variants.
__device__ __forceinline__ bool rot_params(double al, double be, double ga, double tol, double noise, double &c,
                                           double &s, double &t) {
  if (!(al > noise && be > noise && ga * ga > (tol * tol) * (al * be))) return false;
  double d = be - al, g = ga;
  double x = fma(d, d, 4.0 * g * g);
  if (x < 1e-280) {              // tiny columns (exact sweeps, noise = 0): the angle depends on
    const double sc = fast_rcp(fmax(fabs(d), fabs(g)));  // d : g only -- rescale before the
    d *= sc; g *= sc;                                     // flush-to-zero MUFU seed
    x = fma(d, d, 4.0 * g * g);
  }
  const double y = fast_rsqrt(x);
  const double c2 = fma(0.5 * fabs(d), y, 0.5);
  const double z = fast_rsqrt(c2);
  c = c2 * z;
  s = copysign(1.0, d) * g * y * z;
  t = s * z;
  return true;
}

__device__ __forceinline__ void rot_pair(double *ci, double *cj, double *nrm_i, double *nrm_j, int m, double tol,
                                         double noise, int &rot) {
  const int lane = threadIdx.x & 31;
  double ga;
  const bool paired = (m & 1) == 0;        // columns start 16-byte aligned: rows in pairs
  if (paired) {
    const double2 *xi = reinterpret_cast<const double2 *>(ci), *xj = reinterpret_cast<const double2 *>(cj);
    const int n2 = m >> 1;
    double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
    int r = lane;
    for (; r + 32 < n2; r += 64) {          // four independent chains, two 16-byte loads per column
      const double2 x0 = xi[r], y0 = xj[r], x1 = xi[r + 32], y1 = xj[r + 32];
      g0 = fma(x0.x, y0.x, g0); g1 = fma(x0.y, y0.y, g1);
      g2 = fma(x1.x, y1.x, g2); g3 = fma(x1.y, y1.y, g3);
    }
    if (r < n2) { const double2 x0 = xi[r], y0 = xj[r]; g0 = fma(x0.x, y0.x, g0); g1 = fma(x0.y, y0.y, g1); }
    ga = (g0 + g1) + (g2 + g3);
  } else {
    double g0 = 0.0, g1 = 0.0;
    int r = lane;
    for (; r + 32 < m; r += 64) { g0 = fma(ci[r], cj[r], g0); g1 = fma(ci[r + 32], cj[r + 32], g1); }
    if (r < m) g0 = fma(ci[r], cj[r], g0);
    ga = g0 + g1;
  }
  ga = warp_sum(ga);
  const double al = *nrm_i, be = *nrm_j;
  double c, s, t;
  if (rot_params(al, be, ga, tol, noise, c, s, t)) {
    if (paired) {
      double2 *xi = reinterpret_cast<double2 *>(ci), *xj = reinterpret_cast<double2 *>(cj);
      const int n2 = m >> 1;
      for (int r = lane; r < n2; r += 32) {
        const double2 x = xi[r], y = xj[r];
        xi[r] = make_double2(fma(c, x.x, -s * y.x), fma(c, x.y, -s * y.y));
        xj[r] = make_double2(fma(s, x.x, c * y.x), fma(s, x.y, c * y.y));
      }
    } else {
      for (int r = lane; r < m; r += 32) {
        const double x = ci[r], yv = cj[r];
        ci[r] = fma(c, x, -s * yv);
        cj[r] = fma(s, x, c * yv);
      }
    }
    double al2 = fma(-t, ga, al), be2 = fma(t, ga, be);
    __syncwarp();
    if (al2 < 1.5e-8 * al) al2 = col_norm2(ci, m);
    if (be2 < 1.5e-8 * be) be2 = col_norm2(cj, m);
    if (lane == 0) { *nrm_i = al2; *nrm_j = be2; }
    __syncwarp();
    rot = 1;
  }
}

// The WB cross rounds of a block pair with column a of each pair register-resident: warp w
// (< WB) holds column w of block I as R2 double2 per lane (m <= 64 R2, m even) for all WB
// rounds, so each round streams only the partner column WB + (w + sft) % WB through shared
// memory (one read, one write) -- a third of the shared-memory traffic of rot_pair, which
// bounds the rounds (128 B/clk per SM).
#ifndef QTT_COOP_REG
#define QTT_COOP_REG 1
#endif
template <int R2>
__device__ __forceinline__ void cross_rounds_reg(double *S, double *nrmS, int WB, int m, double tol, double noise,
                                                 int &rot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n2 = m >> 1;
  const bool act = warp < WB;
  double2 xa[R2];
  double al = 0.0;
  if (act) {
    const double2 *src = reinterpret_cast<const double2 *>(S + (size_t)warp * m);
#pragma unroll
    for (int k = 0; k < R2; ++k) xa[k] = (lane + 32 * k < n2) ? src[lane + 32 * k] : make_double2(0.0, 0.0);
    al = nrmS[warp];
  }
  for (int sft = 0; sft < WB; ++sft) {
    if (act) {
      const int jb = WB + (warp + sft) % WB;
      double2 *yb = reinterpret_cast<double2 *>(S + (size_t)jb * m);
      double2 yv[R2];
#pragma unroll
      for (int k = 0; k < R2; ++k) yv[k] = (lane + 32 * k < n2) ? yb[lane + 32 * k] : make_double2(0.0, 0.0);
      double g0 = 0.0, g1 = 0.0, g2 = 0.0, g3 = 0.0;
#pragma unroll
      for (int k = 0; k < R2; k += 2) {
        g0 = fma(xa[k].x, yv[k].x, g0); g1 = fma(xa[k].y, yv[k].y, g1);
        if (k + 1 < R2) { g2 = fma(xa[k + 1].x, yv[k + 1].x, g2); g3 = fma(xa[k + 1].y, yv[k + 1].y, g3); }
      }
      const double ga = warp_sum((g0 + g1) + (g2 + g3));
      const double be = nrmS[jb];
      double c, s, t;
      if (rot_params(al, be, ga, tol, noise, c, s, t)) {
        double sa = 0.0, sb = 0.0;
#pragma unroll
        for (int k = 0; k < R2; ++k) {
          const double2 x = xa[k], y = yv[k];
          xa[k] = make_double2(fma(c, x.x, -s * y.x), fma(c, x.y, -s * y.y));
          yv[k] = make_double2(fma(s, x.x, c * y.x), fma(s, x.y, c * y.y));
          if (lane + 32 * k < n2) yb[lane + 32 * k] = yv[k];
        }
        double al2 = fma(-t, ga, al), be2 = fma(t, ga, be);
        if (al2 < 1.5e-8 * al) {          // cancellation: exact refresh from the registers
#pragma unroll
          for (int k = 0; k < R2; ++k) { sa = fma(xa[k].x, xa[k].x, sa); sa = fma(xa[k].y, xa[k].y, sa); }
          al2 = warp_sum(sa);
        }
        if (be2 < 1.5e-8 * be) {
#pragma unroll
          for (int k = 0; k < R2; ++k) { sb = fma(yv[k].x, yv[k].x, sb); sb = fma(yv[k].y, yv[k].y, sb); }
          be2 = warp_sum(sb);
        }
        al = al2;
        if (lane == 0) nrmS[jb] = be2;
        rot = 1;
      }
    }
    __syncthreads();
  }
  if (act) {
    double2 *dst = reinterpret_cast<double2 *>(S + (size_t)warp * m);
#pragma unroll
    for (int k = 0; k < R2; ++k)
      if (lane + 32 * k < n2) dst[lane + 32 * k] = xa[k];
    if (lane == 0) nrmS[warp] = al;
  }
  __syncthreads();
}

// Block I of the Jacobi column partition (columns [I*WB, I*WB+WB) of the column-major m x p
// matrix) is one contiguous run of WB*m doubles: copied with 16-byte accesses, 4 in flight
// per thread, zero beyond column p.
__device__ __forceinline__ void block_copy_in(double *dst, const double *A, int I, int WB, int m, int p) {
  const int nv = max(0, min(WB, p - I * WB));
  const long long n = (long long)nv * m, ntot = (long long)WB * m;
  const double *src = A + (size_t)I * WB * m;
  const int tid = threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const double2 *s2 = reinterpret_cast<const double2 *>(src);
    double2 *d2 = reinterpret_cast<double2 *>(dst);
    const long long n2 = n >> 1;
    long long i = tid;
    for (; i + 3 * kThreads < n2; i += 4 * kThreads) {
      const double2 v0 = __ldcg(s2 + i), v1 = __ldcg(s2 + i + kThreads), v2 = __ldcg(s2 + i + 2 * kThreads),
                    v3 = __ldcg(s2 + i + 3 * kThreads);
      d2[i] = v0; d2[i + kThreads] = v1; d2[i + 2 * kThreads] = v2; d2[i + 3 * kThreads] = v3;
    }
    for (; i < n2; i += kThreads) d2[i] = __ldcg(s2 + i);
    if ((n & 1) && tid == 0) dst[n - 1] = __ldcg(src + n - 1);
  } else {
    for (long long i = tid; i < n; i += kThreads) dst[i] = __ldcg(src + i);
  }
  for (long long i = n + tid; i < ntot; i += kThreads) dst[i] = 0.0;
}

__device__ __forceinline__ void block_copy_out(const double *src, double *A, int I, int WB, int m, int p) {
  const int nv = max(0, min(WB, p - I * WB));
  const long long n = (long long)nv * m;
  double *dst = A + (size_t)I * WB * m;
  const int tid = threadIdx.x;
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
    const double2 *s2 = reinterpret_cast<const double2 *>(src);
    double2 *d2 = reinterpret_cast<double2 *>(dst);
    const long long n2 = n >> 1;
    for (long long i = tid; i < n2; i += kThreads) __stcg(d2 + i, s2[i]);
    if ((n & 1) && tid == 0) __stcg(dst + n - 1, src[n - 1]);
  } else {
    for (long long i = tid; i < n; i += kThreads) __stcg(dst + i, src[i]);
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_jacobi_coop(JacArgs a) {
  extern __shared__ double smj[];
  if (a.skip && *a.skip) return;                        // uniform
  const SiteDims D = *a.dims;
  const int m = D.m, p = D.p, WB = a.WB, g = blockIdx.x, tid = threadIdx.x, warp = tid >> 5;
  const int NB = 2 * ((p + 2 * WB - 1) / (2 * WB));     // even number of blocks
  const double tol = (double)max(m, 1) * DBL_EPSILON;
  double *S = smj;                                      // [2*WB][m]
  double *nrmS = S + (size_t)2 * WB * m;                // [2*WB] column norms of the loaded blocks
  __shared__ int s_rot;
  __shared__ double s_red[kWarps];
  // ||A||_F^2 over CTA slices of the m x p matrix, then an exact power-of-two scale to
  // ||A||_F^2 in [1, 4) (applied at the round-0 block loads, undone at the end): keeps the
  // squares in the rotation test clear of underflow for any input magnitude
  double noise, scale = 1.0;
  {
    const long long n = (long long)m * p;
    double sq = 0.0;
    for (long long i = (long long)g * kThreads + tid; i < n; i += (long long)a.G * kThreads) {
      const double v = __ldcg(a.A + i);
      sq = fma(v, v, sq);
    }
    sq = warp_sum(sq);
    if ((tid & 31) == 0) s_red[warp] = sq;
    __syncthreads();
    if (tid == 0) {
      double b = 0.0;
      for (int w = 0; w < kWarps; ++w) b += s_red[w];
      a.part[g] = b;
    }
    grid_sync(a.bar, a.G, 11);
    double tot = 0.0;
    for (int t = 0; t < a.G; ++t) tot += __ldcg(a.part + t);     // fixed order: deterministic
    if (tot > 0.0 && isfinite(tot)) {
      const int e = -(ilogb(tot) >> 1);
      scale = ldexp(1.0, e);
      tot = ldexp(tot, 2 * e);
    }
    noise = a.noise_ok ? DBL_EPSILON * DBL_EPSILON * tot : 0.0;
  }
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    // 3 rotating flags: slot s%3 collects "rotated in sweep s".  Slot (s+1)%3 was last read at
    // the end of sweep s-2 and every CTA has passed the barriers of sweep s-1 since, so it is
    // cleared here (for sweep s+1) without racing a reader.
    if (g == 0 && tid == 0) a.flags[(sweep + 1) % 3] = 0;
    int rot = 0;
    for (int r = 0; r < NB - 1; ++r) {
      const int R = sweep * (NB - 1) + r;          // global block round
      for (int t = g; t < NB / 2; t += a.G) {
        const int I = (t == 0) ? 0 : 1 + (t - 1 + r) % (NB - 1);
        const int J = 1 + (NB - 2 - t + r) % (NB - 1);
        // dataflow instead of a grid barrier per block round: wait until both blocks carry the
        // result of round R - 1 (their producers pulled earlier rounds, so no deadlock)
        if (tid == 0) {
          int v;
          long long spins = 0;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(a.ver + I) : "memory");
            if (v >= R) asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(a.ver + J) : "memory");
            if (v < R) __nanosleep(32);
            if (++spins > (1LL << 26)) { atomicOr(a.status, ST_NOCONV); break; }   // report, do not hang
          } while (v < R);
          __threadfence();
        }
        __syncthreads();
        // load the two blocks (zero columns beyond p)
        block_copy_in(S, a.A, I, WB, m, p);
        block_copy_in(S + (size_t)WB * m, a.A, J, WB, m, p);
        if (sweep == 0 && r == 0 && scale != 1.0) {             // every block is loaded once in round 0
          __syncthreads();
          for (int i = tid; i < 2 * WB * m; i += kThreads) S[i] *= scale;
        }
        __syncthreads();
        if (r == 0) {                     // exact norms once per sweep (every block is in round 0)
          for (int c = warp; c < 2 * WB; c += kWarps) {
            const double v = col_norm2(S + (size_t)c * m, m);
            if ((tid & 31) == 0) nrmS[c] = v;
          }
        } else if (tid < 2 * WB) {        // otherwise the norms carried with the columns
          const int col = (tid < WB) ? I * WB + tid : J * WB + tid - WB;
          nrmS[tid] = (col < p) ? __ldcg(a.nrm + col) : 0.0;
        }
        __syncthreads();
        if (r == 0 && WB > 1) {           // intra-block pairs (circle method on WB players)
          for (int u = 0; u < WB - 1; ++u) {
            for (int pr = warp; pr < WB; pr += kWarps) {
              const int h = WB / 2, tt = pr % h, base = (pr < h) ? 0 : WB;
              const int k1 = tt, k2 = WB - 1 - tt;
              const int i = base + ((k1 == 0) ? 0 : 1 + (k1 - 1 + u) % (WB - 1));
              const int j = base + ((k2 == 0) ? 0 : 1 + (k2 - 1 + u) % (WB - 1));
              rot_pair(S + (size_t)i * m, S + (size_t)j * m, nrmS + i, nrmS + j, m, tol, noise, rot);
            }
            __syncthreads();
          }
        }
        // cross pairs (a, WB + (a+sft)%WB), sft = 0..WB-1
        const bool regs = QTT_COOP_REG && (m & 1) == 0 && WB <= kWarps;
        if (regs && m <= 256) cross_rounds_reg<4>(S, nrmS, WB, m, tol, noise, rot);
        else if (regs && m <= 512) cross_rounds_reg<8>(S, nrmS, WB, m, tol, noise, rot);
        // (m <= 1024 in registers, R2 = 16, needs all 255 registers and measured slower on cfg4)
        else
          for (int sft = 0; sft < WB; ++sft) {
            for (int pr = warp; pr < WB; pr += kWarps)
              rot_pair(S + (size_t)pr * m, S + (size_t)(WB + (pr + sft) % WB) * m, nrmS + pr,
                       nrmS + WB + (pr + sft) % WB, m, tol, noise, rot);
            __syncthreads();
          }
        block_copy_out(S, a.A, I, WB, m, p);
        block_copy_out(S + (size_t)WB * m, a.A, J, WB, m, p);
        if (tid < 2 * WB) {
          const int col = (tid < WB) ? I * WB + tid : J * WB + tid - WB;
          if (col < p) __stcg(a.nrm + col, nrmS[tid]);
        }
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(a.ver + I), "r"(R + 1) : "memory");
          asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(a.ver + J), "r"(R + 1) : "memory");
        }
      }
    }
    if (tid == 0) s_rot = 0;
    __syncthreads();
    if (rot) s_rot = 1;
    __syncthreads();
    if (tid == 0 && s_rot) atomicOr(a.flags + (sweep % 3), 1);
    grid_sync(a.bar, a.G, 12);
    const int any = *((volatile int *)(a.flags + (sweep % 3)));
    if (!any) { ++sweep; break; }
  }
  if (scale != 1.0) {              // the last grid barrier ordered every block store before this
    const double inv = 1.0 / scale;
    const long long n = (long long)m * p;
    for (long long i = (long long)g * kThreads + tid; i < n; i += (long long)a.G * kThreads)
      __stcg(a.A + i, __ldcg(a.A + i) * inv);
  }
  if (g == 0 && tid == 0) {
    *a.sweeps_out = sweep;
    if (sweep >= 60) atomicOr(a.status, ST_NOCONV);
  }
}

// ------------------------------------------------------------------ a5/a6: finish

struct FinishArgs {
  SiteDims *dims;
  const double *A;        // m x p column-major
  double *Cq;             // output core slot: (chi, d, k) = m x k row-major
  int *yr_next;           // out_ranks[b][q+1]
  double *delta2;         // &delta2[b*L+q]
  double *sigma;          // &sigma[(b*(L-1)+q)*stride] or NULL
  int sigma_stride;
  double *s2;             // scratch [pcap]
  int *perm;              // scratch [pcap]
  double eps;
  int max_rank;
  int *status;
  GemmSpec *carry;        // spec[2]: G' = Cq^T T
  const double *T;
  double *Gout;
  const int *skip;        // non-NULL and set: the site was done by CholeskyQR2 (a1 sweeps)
};

__global__ void __launch_bounds__(kThreads, 1) k_finish(FinishArgs a) {
  __shared__ double sc[4];
  if (a.skip && *a.skip) return;
  SiteDims D = *a.dims;
  const int m = D.m, p = D.p, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = warp; j < p; j += kWarps) {
    double s = 0.0;
    for (int r = lane; r < m; r += 32) { const double v = a.A[(size_t)j * m + r]; s = fma(v, v, s); }
    s = warp_sum(s);
    if (lane == 0) {
      if (!isfinite(s)) { atomicOr(a.status, ST_NONFINITE); s = 0.0; }
      a.s2[j] = s;
    }
  }
  __syncthreads();
  for (int j = tid; j < p; j += kThreads) {
    const double sj = a.s2[j];
    int rank = 0;
    for (int l = 0; l < p; ++l) rank += (a.s2[l] > sj) || (a.s2[l] == sj && l < j);
    a.perm[rank] = j;
  }
  __syncthreads();
  if (tid == 0) {
    double acc = 0.0, tot = 0.0;
    for (int jj = p - 1; jj >= 0; --jj) tot += a.s2[a.perm[jj]];
    const double tau = a.eps * a.eps * tot;
    int k = p;
    for (int kk = p - 1; kk >= 1; --kk) {       // tail[kk] = sum_{j>=kk} s_j^2 (smallest first)
      acc += a.s2[a.perm[kk]];
      if (acc <= tau) k = kk; else break;
    }
    // recompute tail[k] in the same order as the oracle
    double tail = 0.0;
    for (int jj = p - 1; jj >= k; --jj) tail += a.s2[a.perm[jj]];
    const int kc = (a.max_rank > 0 && D.kcap > 0) ? min(a.max_rank, D.kcap) : (a.max_rank > 0 ? a.max_rank : D.kcap);
    if (kc > 0 && k > kc) {
      k = kc;
      tail = 0.0;
      for (int jj = p - 1; jj >= k; --jj) tail += a.s2[a.perm[jj]];
    }
    if (tot == 0.0) { k = 1; tail = 0.0; }
    k = max(k, 1);
    sc[0] = (double)k; sc[1] = tail;
    *a.yr_next = k;
    *a.delta2 = tail;
    a.dims->k = k;
    GemmSpec gc{};
    gc.M = k; gc.N = D.n; gc.K = m; gc.nz1 = 1; gc.nz2 = 1;
    gc.A = a.Cq; gc.sam = 1; gc.sak = k;
    gc.B = a.T; gc.sbk = D.n; gc.sbn = 1;
    gc.C = a.Gout; gc.scm = D.n; gc.scn = 1;
    *a.carry = gc;
  }
  __syncthreads();
  const int k = (int)sc[0];
  for (long long idx = tid; idx < (long long)m * k; idx += kThreads) {
    const int row = (int)(idx / k), kk = (int)(idx % k);
    const int j = a.perm[kk];
    const double s2 = a.s2[j];
    a.Cq[idx] = (s2 > 0.0) ? a.A[(size_t)j * m + row] / sqrt(s2) : (row == kk ? 1.0 : 0.0);
  }
  if (a.sigma)
    for (int jj = tid; jj < a.sigma_stride; jj += kThreads) a.sigma[jj] = (jj < p) ? sqrt(a.s2[a.perm[jj]]) : 0.0;
}

__global__ void k_last(const SiteDims *dims, const double *T, double *Cq, double *norm2, double *delta2, int *yr_L,
                       int *status) {
  __shared__ double red[kWarps];
  const SiteDims D = *dims;
  double s = 0.0;
  for (int i = threadIdx.x; i < D.m; i += kThreads) { const double v = T[i]; Cq[i] = v; s = fma(v, v, s); }
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    *norm2 = s; *delta2 = 0.0; *yr_L = 1;
    if (!isfinite(s)) atomicOr(status, ST_NONFINITE);
  }
}

// ------------------------------------------------------------------ mirror (large a1)

struct MirrorL {
  int L, dm[64];
  int cap_src[65];
  const double *src[64];
  long long src_bs;        // unused (single member)
  const int *src_ranks;    // device [L+1] or NULL
  double *dst[64];
  int pad;
  int *dst_ranks;
};

__global__ void k_mirror_l(MirrorL a) {
  const int qd = blockIdx.x, qs = a.L - 1 - qd;
  const int rl = a.src_ranks ? a.src_ranks[qs] : a.cap_src[qs];
  const int rr = a.src_ranks ? a.src_ranks[qs + 1] : a.cap_src[qs + 1];
  const int d = a.dm[qs];
  const double *s = a.src[qs];
  double *t = a.dst[qd];
  if (a.pad) {
    const int cl = a.cap_src[qs + 1], cr = a.cap_src[qs];
    const long long n = (long long)cl * d * cr;
    for (long long idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const int aa = (int)(idx % cr);
      const long long t1 = idx / cr;
      const int i = (int)(t1 % d), ap = (int)(t1 / d);
      t[idx] = (ap < rr && aa < rl) ? s[((size_t)aa * d + i) * rr + ap] : 0.0;
    }
  } else {
    const long long n = (long long)rr * d * rl;
    for (long long idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const int aa = (int)(idx % rl);
      const long long t1 = idx / rl;
      const int i = (int)(t1 % d), ap = (int)(t1 / d);
      t[idx] = s[((size_t)aa * d + i) * rr + ap];
    }
    if (threadIdx.x == 0) {
      a.dst_ranks[qd + 1] = rl;
      if (qd == 0) a.dst_ranks[0] = rr;
    }
  }
}

// ------------------------------------------------------------------ host: one sweep

struct SweepBufs {
  double *G, *X, *T, *Tw, *A, *part, *wtot, *gram, *bc, *s2;
  int *perm, *flags, *ver, *sweeps_scratch;
  GridBar *bar;
  SiteDims *dims;
  GemmSpec *spec;
};

static int g_sms = 0;

static qtt_status_t sweep_caps(int L, const std::vector<int> &d, const std::vector<int> &dj, const std::vector<int> &xr,
                               const std::vector<int> &orr, const std::vector<int> &cap, int kind, long long &mcap,
                               long long &ncap, long long &gcap, long long &xcap, long long &tcap, long long &acap,
                               long long &pcap) {
  mcap = ncap = gcap = xcap = tcap = acap = pcap = 1;
  for (int q = 0; q < L; ++q) {
    const long long m = (long long)cap[q] * d[q];
    const long long n = (long long)orr[q + 1] * xr[q + 1];
    mcap = std::max(mcap, m); ncap = std::max(ncap, n);
    gcap = std::max(gcap, (long long)cap[q] * orr[q] * xr[q]);
    gcap = std::max(gcap, (long long)cap[q + 1] * n);
    const long long xe = (kind == MATVEC) ? (long long)cap[q] * orr[q] * dj[q] * xr[q + 1]
                                          : (kind == HADAMARD ? (long long)cap[q] * orr[q] * d[q] * xr[q + 1] : 1);
    xcap = std::max(xcap, xe);
    tcap = std::max(tcap, m * n);
    acap = std::max(acap, m * std::min(m, n));
    pcap = std::max(pcap, std::min(m, n));
  }
  return QTT_OK;
}

struct SweepPlan {
  long long mcap, ncap, gcap, xcap, tcap, acap, pcap;
  int Gqr, RB, Gjac, WB;
  size_t qr_smem, jac_smem;
  size_t off_G, off_X, off_T, off_Tw, off_A, off_part, off_wtot, off_gram, off_bc, off_s2, off_perm, off_flags,
      off_ver, off_sw, off_bar, off_dims, off_spec, total;
  // tall sites: Householder QR first, explicit Q applied to U_R
  int tq;
  size_t off_tqDims, off_tqI, off_tqR, off_tqTau;
  // CholeskyQR2 (cholqr.cuh) for the wide sites
  int cq, cq_S, cq_nblk, cq_G;
  size_t off_cqP, off_cqR1, off_cqR2, off_cqRinv, off_cqDinv, off_cqI, off_cqDev, off_cqSpec;
};

constexpr int kCqMinRows = 64;        // smaller site matrices keep the Householder QR (cheap there)

static qtt_status_t plan_sweep(int L, const std::vector<int> &d, const std::vector<int> &dj, const std::vector<int> &xr,
                               const std::vector<int> &orr, const std::vector<int> &cap, int kind, SweepPlan &P) {
  sweep_caps(L, d, dj, xr, orr, cap, kind, P.mcap, P.ncap, P.gcap, P.xcap, P.tcap, P.acap, P.pcap);
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  // QR: rows of T^H per CTA <= kQrRowsMax, >= 32
  P.Gqr = (int)std::min<long long>(g_sms, std::max<long long>(1, (P.ncap + 31) / 32));
  P.RB = (int)((P.ncap + P.Gqr - 1) / P.Gqr);
  P.RB = ((P.RB + 31) / 32) * 32;
  while (P.RB > kQrRowsMax) { set_error("large path: n = %lld too large", P.ncap); return QTT_EUNSUPPORTED; }
  P.qr_smem = sizeof(double) * ((size_t)kNb * P.RB + 32 + kNb * kNb + 2 * kNb + kNb * 64);
  // Jacobi: blocks of WB = kWarps columns -- every warp has a pair in each cross round, and a
  // block round (dataflow wait + block copies) is amortised over WB rounds (measured: cfg2
  // 134 -> 101 ms against ~64 blocks of 4; cfg3 already had WB = 8), capped by smem
  int WB = kWarps;
  if (const char *e = getenv("QTT_COOP_WB")) {         // A/B knob (diagnostics): a power of two <= 64
    const int w = std::max(1, std::min(64, atoi(e)));
    WB = 1;
    while (2 * WB <= w) WB *= 2;
  }
  while (WB > 1 && 2 * WB * (P.mcap + 1) * 8 > 200 * 1024) WB /= 2;
  if (2 * WB * (P.mcap + 1) * 8 > 200 * 1024) { set_error("large path: m = %lld too large", P.mcap); return QTT_EUNSUPPORTED; }
  P.WB = WB;
  P.Gjac = (int)std::min<long long>(g_sms, std::max<long long>(1, (P.pcap + 2 * WB - 1) / (2 * WB)));
  P.jac_smem = sizeof(double) * (2 * WB * P.mcap + 2 * WB);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  P.off_G = take(8 * P.gcap);
  P.off_X = take(8 * P.xcap);
  P.off_T = take(8 * P.tcap);
  P.off_Tw = take(8 * P.tcap);
  P.off_A = take(8 * P.acap);
  // (the tall-site QR / Q apply run on up to ceil(mcap / 32) CTAs)
  const size_t Gpart = std::max<size_t>(P.Gqr, std::min<size_t>(g_sms, (P.mcap + 31) / 32));
  P.off_part = take(8 * (Gpart * kNb * P.mcap + Gpart * kNb * kNb + 16 + g_sms));
  P.off_wtot = take(8 * (size_t)kNb * P.mcap);
  P.off_gram = take(8 * kNb * kNb);
  P.off_bc = take(8 * 64);
  P.off_s2 = take(8 * P.pcap);
  P.off_perm = take(4 * P.pcap);
  P.off_flags = take(4 * 4);
  P.off_ver = take(4 * ((size_t)P.pcap + 2));
  P.off_sw = take(4 * 4);
  P.off_bar = take(sizeof(GridBar) * 2);
  P.off_dims = take(sizeof(SiteDims));
  P.off_spec = take(sizeof(GemmSpec) * 3);
  P.tq = (P.mcap >= 64 && getenv("QTT_NO_TALLQR") == nullptr) ? 1 : 0;
  if (P.tq) {
    P.off_tqDims = take(sizeof(SiteDims) * 3);
    P.off_tqI = take(32);                       // tq, ntq, (pad), the QR's scale (double at +16)
    P.off_tqR = take(8 * (size_t)P.pcap * P.pcap);
    P.off_tqTau = take(8 * (size_t)P.pcap);
  }
  // CholeskyQR2: only when some site can be wide with m >= kCqMinRows
  P.cq = (P.mcap >= kCqMinRows && getenv("QTT_NO_CHOLQR") == nullptr) ? 1 : 0;
  if (P.cq) {
    const long long tt = (P.mcap + dgemm::TM - 1) / dgemm::TM;
    const long long tiles = tt * (tt + 1) / 2;                 // the Gram GEMMs compute upper tiles only
    P.cq_S = (int)std::max<long long>(1, std::min<long long>(16, g_sms / tiles));
    P.cq_nblk = (int)((P.mcap + kCholNb - 1) / kCholNb);
    // the Cholesky's trailing work is small (<= nblk^2/2 tiles of 32^3 per block row): a few CTAs
    // keep its 2 nblk grid barriers short
    P.cq_G = (int)std::min<long long>(32, std::max<long long>(1, (long long)P.cq_nblk * (P.cq_nblk + 1) / 2));
    const size_t m2 = (size_t)P.mcap * P.mcap;
    P.off_cqP = take(8 * m2 * P.cq_S);
    P.off_cqR1 = take(8 * m2);
    P.off_cqR2 = take(8 * m2);
    P.off_cqRinv = take(8 * m2);
    P.off_cqDinv = take(8 * (size_t)P.cq_nblk * kCholNb * kCholNb);
    P.off_cqI = take(4 * 4);
    P.off_cqDev = take(8 * 2);
    P.off_cqSpec = take(sizeof(GemmSpec) * 9);     // [0..3] wide, [4..8] tall
  }
  P.total = off;
  return QTT_OK;
}

static qtt_status_t coop_launch(const void *fn, int grid, size_t smem, void *args, cudaStream_t s) {
  void *kargs[] = {args};
  QTT_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), kargs, smem, s));
  return QTT_OK;
}

__global__ void k_site0_init(double *G, int *yr) {
  if (threadIdx.x == 0) { G[0] = 1.0; yr[0] = 1; }
}

// One member's sweep a2..a7.  Xq/Oq/Wop per site point at this member's workspace operand
// copies; xr/orr/yr are this member's device rank rows; orig_xr/orig_or are capacities.
struct SweepIO {
  int L, kind;
  std::vector<int> d, dj, cap, xcap_r, ocap_r;     // digit sizes, output caps, operand rank caps
  std::vector<const double *> Xq, Oq;              // Oq: Hadamard second state / MPO cores
  const int *xr, *orr;
  int *yr;
  std::vector<double *> Cq;
  double *delta2, *norm2, *sigma;
  int sigma_stride;
  int *sweeps, *status;
  double eps;
  int max_rank;
  bool tf32 = false;                               // contraction GEMMs as 3xTF32 (fp32 variant)
};

static qtt_status_t run_sweep(const SweepIO &io, const SweepPlan &P, char *ws, cudaStream_t s) {
  const int L = io.L, kind = io.kind;
  SweepBufs Bf;
  Bf.G = (double *)(ws + P.off_G); Bf.X = (double *)(ws + P.off_X); Bf.T = (double *)(ws + P.off_T);
  Bf.Tw = (double *)(ws + P.off_Tw); Bf.A = (double *)(ws + P.off_A); Bf.part = (double *)(ws + P.off_part);
  Bf.wtot = (double *)(ws + P.off_wtot); Bf.gram = (double *)(ws + P.off_gram); Bf.bc = (double *)(ws + P.off_bc);
  Bf.s2 = (double *)(ws + P.off_s2); Bf.perm = (int *)(ws + P.off_perm); Bf.flags = (int *)(ws + P.off_flags);
  Bf.ver = (int *)(ws + P.off_ver);
  Bf.sweeps_scratch = (int *)(ws + P.off_sw); Bf.bar = (GridBar *)(ws + P.off_bar);
  Bf.dims = (SiteDims *)(ws + P.off_dims); Bf.spec = (GemmSpec *)(ws + P.off_spec);
  {  // dynamic-smem opt-in on the current device, every call (per-device setting; cheap, thread-safe)
    QTT_CUDA_TRY(cudaFuncSetAttribute(k_qr_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    QTT_CUDA_TRY(cudaFuncSetAttribute(k_qapply_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    QTT_CUDA_TRY(cudaFuncSetAttribute(k_jacobi_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    QTT_CUDA_TRY(cudaFuncSetAttribute(k_gemm_dmma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)dgemm::SMEM_BYTES));
    QTT_CUDA_TRY(cudaFuncSetAttribute(k_gemm_dmma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)dgemm::SMEM_BYTES));
    QTT_CUDA_TRY(cudaFuncSetAttribute(k_gemm_dmma<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)dgemm::SMEM_BYTES));
    QTT_CUDA_TRY(cudaFuncSetAttribute(k_gemm_tf32<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)tf32g::SMEM_BYTES));
    QTT_CUDA_TRY(cudaFuncSetAttribute(k_gemm_tf32<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)tf32g::SMEM_BYTES));
  }
  QTT_CUDA_TRY(cudaMemsetAsync(Bf.bar, 0, sizeof(GridBar) * 2, s));
  k_site0_init<<<1, 32, 0, s>>>(Bf.G, io.yr);
  QTT_CUDA_TRY(cudaGetLastError());
  for (int q = 0; q < L; ++q) {
    const long long w = (kind == TRUNCATE) ? 1 : io.ocap_r[q], w2 = (kind == TRUNCATE) ? 1 : io.ocap_r[q + 1];
    const long long m_cap = (long long)io.cap[q] * io.d[q];
    const long long n_cap = w2 * io.xcap_r[q + 1];
    PlanArgs pa;
    pa.q = q; pa.L = L; pa.kind = kind; pa.d = io.d[q]; pa.dj = io.dj[q];
    pa.xr = io.xr; pa.orr = io.orr; pa.yr = io.yr;
    pa.Xq = io.Xq[q]; pa.Oq = (kind == TRUNCATE) ? nullptr : io.Oq[q];
    pa.G = Bf.G; pa.X = Bf.X; pa.T = Bf.T; pa.Cq = io.Cq[q];
    pa.dims = Bf.dims; pa.spec = Bf.spec;
    k_plan<<<1, 32, 0, s>>>(pa);
    QTT_CUDA_TRY(cudaGetLastError());
    // a2: state GEMM (M <= cap*w, N <= (dj|d)*r2)
    const long long g0M = (long long)io.cap[q] * w;
    const long long g0N = (long long)((kind == MATVEC) ? io.dj[q] : io.d[q]) * io.xcap_r[q + 1];
    launch_gemm_spec(Bf.spec + 0, g0M, g0N, 1, 1, true, io.tf32, s);
    QTT_CUDA_TRY(cudaGetLastError());
    const unsigned ew_grid = (unsigned)std::min<long long>((m_cap * n_cap + kThreads - 1) / kThreads, 8192);
    if (kind == MATVEC) {
      k_mpo_apply<<<ew_grid, kThreads, 0, s>>>(Bf.dims, Bf.X, io.Oq[q], Bf.T);
      QTT_CUDA_TRY(cudaGetLastError());
    } else if (kind == HADAMARD) {
      launch_gemm_spec(Bf.spec + 1, w2, io.xcap_r[q + 1], io.cap[q], io.d[q], false, io.tf32, s);
      QTT_CUDA_TRY(cudaGetLastError());
    }
    if (q == L - 1) {                                                  // a7
      k_last<<<1, kThreads, 0, s>>>(Bf.dims, Bf.T, io.Cq[q], io.norm2, io.delta2 + q, io.yr + L, io.status);
      QTT_CUDA_TRY(cudaGetLastError());
      if (io.sweeps) QTT_CUDA_TRY(cudaMemsetAsync(io.sweeps + q, 0, sizeof(int), s));
      break;
    }
    // a1 sweeps (truncate, eps = 0): tall sites orthonormalised by CholeskyQR2 with Q explicit
    int *cqt_ok = nullptr;
    if (P.cq && kind == TRUNCATE && io.eps == 0.0 && io.max_rank <= 0 && !io.sigma) {
      cqt_ok = (int *)(ws + P.off_cqI) + 2;
      int *cqt_n = cqt_ok + 1;
      double *cq_dev = (double *)(ws + P.off_cqDev) + 1;
      GemmSpec *cs = (GemmSpec *)(ws + P.off_cqSpec) + 4;
      double *R1 = (double *)(ws + P.off_cqR1), *R2 = (double *)(ws + P.off_cqR2);
      double *Rinv = (double *)(ws + P.off_cqRinv), *Dinv = (double *)(ws + P.off_cqDinv);
      double *Pp = (double *)(ws + P.off_cqP);
      const long long m2 = P.mcap * P.mcap;
      CqtPlanArgs ta{Bf.dims, P.cq_S, 32, Bf.T, Bf.Tw, Pp, Rinv, R1, R2, io.Cq[q], Bf.G, m2, cs, cqt_ok, cqt_n, cq_dev};
      k_cqt_plan<<<1, 32, 0, s>>>(ta);
      QTT_CUDA_TRY(cudaGetLastError());
      const long long nc = std::min<long long>(m_cap, n_cap);
      const long long tn = (nc + dgemm::TM - 1) / dgemm::TM;
      const unsigned rgrid = (unsigned)std::min<long long>((nc * nc + 255) / 256, 2048);
      auto gram = [&](int which, double *Wout, double *dev) -> qtt_status_t {
        k_gemm_dmma<false, false><<<dim3((unsigned)(tn * tn), 1, (unsigned)P.cq_S), 256, dgemm::SMEM_BYTES, s>>>(
            cs + which, (int)tn, 1);
        QTT_CUDA_TRY(cudaGetLastError());
        RedArgs ra{Pp, m2, P.cq_S, cqt_n, cqt_ok, Wout, dev};
        k_gram_reduce<<<rgrid, kThreads, 0, s>>>(ra);
        QTT_CUDA_TRY(cudaGetLastError());
        return QTT_OK;
      };
      auto chol = [&](double *W, double *dev) -> qtt_status_t {
        CholArgs ch{W, Dinv, cqt_n, cqt_ok, dev, 0.25, Bf.bar, P.cq_G};
        return coop_launch((const void *)k_chol_coop, P.cq_G, 0, &ch, s);
      };
      auto trinv = [&](double *R) -> qtt_status_t {
        TrinvArgs tv{R, Dinv, Rinv, cqt_n, cqt_ok};
        k_trinv<<<(unsigned)P.cq_nblk, kThreads, 0, s>>>(tv);
        QTT_CUDA_TRY(cudaGetLastError());
        return QTT_OK;
      };
      qtt_status_t st = gram(0, R1, nullptr);                          // W = T^T T
      if (st == QTT_OK) st = chol(R1, nullptr);
      if (st == QTT_OK) { k_cq_gate<<<1, 32, 0, s>>>(cqt_ok, cs, 1, 5); st = trinv(R1); }
      if (st != QTT_OK) return st;
      launch_gemm_spec(cs + 1, m_cap, nc, 1, 1, true, false, s);        // Q1 = T Rinv1 -> Tw
      QTT_CUDA_TRY(cudaGetLastError());
      st = gram(2, R2, cq_dev);                                        // W2 = Q1^T Q1
      if (st == QTT_OK) st = chol(R2, cq_dev);
      if (st == QTT_OK) { k_cq_gate<<<1, 32, 0, s>>>(cqt_ok, cs, 3, 5); st = trinv(R2); }
      if (st != QTT_OK) return st;
      launch_gemm_spec(cs + 3, m_cap, nc, 1, 1, true, false, s);        // Q = Q1 Rinv2 -> C_q
      QTT_CUDA_TRY(cudaGetLastError());
      k_gemm_dmma<true, false><<<dim3((unsigned)(tn * tn), 1, 1), 256, dgemm::SMEM_BYTES, s>>>(cs + 4, (int)tn, 1);
      QTT_CUDA_TRY(cudaGetLastError());                                // R = R2 R1 -> carry G
    }
    // a3: CholeskyQR2 when the gate accepts the site, else the Householder QR
    int *cq_ok = nullptr;
    if (P.cq) {
      cq_ok = (int *)(ws + P.off_cqI);
      int *cq_m = cq_ok + 1;
      double *cq_dev = (double *)(ws + P.off_cqDev);
      GemmSpec *cs = (GemmSpec *)(ws + P.off_cqSpec);
      double *R1 = (double *)(ws + P.off_cqR1), *R2 = (double *)(ws + P.off_cqR2);
      double *Rinv = (double *)(ws + P.off_cqRinv), *Dinv = (double *)(ws + P.off_cqDinv);
      double *Pp = (double *)(ws + P.off_cqP);
      const long long m2 = P.mcap * P.mcap;
      CqPlanArgs ca{Bf.dims, P.cq_S, kCqMinRows, Bf.T, Bf.Tw, Pp, Rinv, R1, R2, Bf.A, m2, cs, cq_ok, cq_m, cq_dev};
      k_cq_plan<<<1, 32, 0, s>>>(ca);
      QTT_CUDA_TRY(cudaGetLastError());
      const long long mc = std::min<long long>(m_cap, n_cap);
      const long long tm = (mc + dgemm::TM - 1) / dgemm::TM, tn = tm;
      const unsigned rgrid = (unsigned)std::min<long long>((mc * mc + 255) / 256, 2048);
      auto gram = [&](int which, double *Wout, double *dev) -> qtt_status_t {
        k_gemm_dmma<true, true><<<dim3((unsigned)(tm * tn), 1, (unsigned)P.cq_S), 256, dgemm::SMEM_BYTES, s>>>(
            cs + which, (int)tn, 1);
        QTT_CUDA_TRY(cudaGetLastError());
        RedArgs ra{Pp, m2, P.cq_S, cq_m, cq_ok, Wout, dev};
        k_gram_reduce<<<rgrid, kThreads, 0, s>>>(ra);
        QTT_CUDA_TRY(cudaGetLastError());
        return QTT_OK;
      };
      auto chol = [&](double *W, double *dev) -> qtt_status_t {
        CholArgs ch{W, Dinv, cq_m, cq_ok, dev, 0.25, Bf.bar, P.cq_G};
        return coop_launch((const void *)k_chol_coop, P.cq_G, 0, &ch, s);
      };
      qtt_status_t st = gram(0, R1, nullptr);                          // W = T T^T
      if (st == QTT_OK) st = chol(R1, nullptr);                        // R1
      if (st != QTT_OK) return st;
      k_cq_gate<<<1, 32, 0, s>>>(cq_ok, cs, 1);
      TrinvArgs ta{R1, Dinv, Rinv, cq_m, cq_ok};
      k_trinv<<<(unsigned)P.cq_nblk, kThreads, 0, s>>>(ta);            // Rinv = R1^-1
      QTT_CUDA_TRY(cudaGetLastError());
      launch_gemm_spec(cs + 1, mc, n_cap, 1, 1, false, false, s);      // Q1^T = Rinv^T T -> Tw
      QTT_CUDA_TRY(cudaGetLastError());
      st = gram(2, R2, cq_dev);                                        // W2 = Q1^T Q1, |W2 - I|_F^2
      if (st == QTT_OK) st = chol(R2, cq_dev);                         // R2 (gate |W2 - I|_F <= 1/2)
      if (st != QTT_OK) return st;
      k_cq_gate<<<1, 32, 0, s>>>(cq_ok, cs, 3);
      k_gemm_dmma<true, false><<<dim3((unsigned)(tm * tn), 1, 1), 256, dgemm::SMEM_BYTES, s>>>(cs + 3, (int)tn, 1);
      QTT_CUDA_TRY(cudaGetLastError());                                // R = R2 R1 -> A
    }
    k_copy_T<<<ew_grid, kThreads, 0, s>>>(Bf.dims, Bf.T, Bf.Tw, Bf.A, cq_ok, cqt_ok);
    QTT_CUDA_TRY(cudaGetLastError());
    {
      QrArgs qa;
      qa.dims = Bf.dims; qa.Tw = Bf.Tw; qa.Rout = Bf.A; qa.part = Bf.part; qa.wtot = Bf.wtot; qa.gram = Bf.gram;
      qa.bc = Bf.bc; qa.bar = Bf.bar; qa.G = P.Gqr; qa.RB = P.RB; qa.mcap = (int)P.mcap; qa.skip = cq_ok; qa.tau_out = nullptr;
      qtt_status_t st = coop_launch((const void *)k_qr_coop, P.Gqr, P.qr_smem, &qa, s);
      if (st != QTT_OK) return st;
    }
    // tall sites (m >= 2n): Householder QR of T first; the Jacobi / finish then see R's dims
    SiteDims *dims_j = Bf.dims;
    int *tq = nullptr, tq_G = 0, tq_RB = 0;
    size_t tq_smem = 0;
    const bool tq_cand = P.tq && m_cap >= 2 * n_cap && n_cap >= 64 && m_cap >= 1024;
    if (tq_cand) {
      dims_j = (SiteDims *)(ws + P.off_tqDims);
      SiteDims *dims_t = dims_j + 1;
      tq = (int *)(ws + P.off_tqI);
      int *ntq = tq + 1;
      double *Rt = (double *)(ws + P.off_tqR), *tauv = (double *)(ws + P.off_tqTau);
      SiteDims *dims_2 = dims_j + 2;
      TqPlanArgs tp{Bf.dims, dims_j, dims_t, dims_2, tq, ntq, cqt_ok};
      k_tq_plan<<<1, 32, 0, s>>>(tp);
      double *tq_scale = (double *)(ws + P.off_tqI + 16);
      k_tq_sq<<<g_sms, kThreads, 0, s>>>(Bf.dims, tq, Bf.T, Bf.part);
      k_tq_copy<<<ew_grid, kThreads, 0, s>>>(Bf.dims, tq, Bf.T, Bf.part, g_sms, Bf.Tw, tq_scale);
      QTT_CUDA_TRY(cudaGetLastError());
      QrArgs qt;
      qt.dims = dims_t; qt.Tw = Bf.Tw; qt.Rout = Rt; qt.part = Bf.part; qt.wtot = Bf.wtot; qt.gram = Bf.gram;
      // the QR's grid from this site's rows (fewer CTAs in each column step's barrier)
      tq_G = (int)std::min<long long>(g_sms, (m_cap + 31) / 32);
      tq_RB = (int)(((m_cap + tq_G - 1) / tq_G + 31) / 32 * 32);
      tq_smem = sizeof(double) * ((size_t)kNb * tq_RB + 32 + kNb * kNb + 2 * kNb + kNb * 64);
      qt.bc = Bf.bc; qt.bar = Bf.bar; qt.G = tq_G; qt.RB = tq_RB; qt.mcap = (int)P.mcap; qt.skip = ntq;
      qt.tau_out = tauv;
      qtt_status_t st = coop_launch((const void *)k_qr_coop, tq_G, tq_smem, &qt, s);
      if (st != QTT_OK) return st;
      // second QR, of R1^T (its columns are R1's rows, i.e. Rt as k_qr_coop's row-major input):
      // R1^T = Q2 R2, so R1 = R2^T Q2^T and the Jacobi on R2^T's columns yields R1's -- hence
      // (after Q1) T's -- left singular vectors with no rotation accumulation, in about half the
      // sweeps of the Jacobi on R1 (measured on cfg4's 2560 x 1000 site: 13 against 27)
      const bool qr2 = getenv("QTT_TQ_QR1") == nullptr;
      if (qr2) {
        QrArgs q2 = qt;
        const long long n2 = n_cap;
        q2.dims = dims_2; q2.Tw = Rt; q2.Rout = Bf.A; q2.tau_out = nullptr;
        q2.G = (int)std::min<long long>(g_sms, (n2 + 31) / 32);
        q2.RB = (int)(((n2 + q2.G - 1) / q2.G + 31) / 32 * 32);
        const size_t sm2 = sizeof(double) * ((size_t)kNb * q2.RB + 32 + kNb * kNb + 2 * kNb + kNb * 64);
        st = coop_launch((const void *)k_qr_coop, q2.G, sm2, &q2, s);
        if (st != QTT_OK) return st;
      }
      k_tq_toA<<<(unsigned)std::min<long long>((P.pcap * P.pcap + 255) / 256, 4096), 256, 0, s>>>(
          Bf.dims, tq, qr2 ? Bf.A : Rt, tq_scale, Bf.A, qr2 ? 1 : 0);
      QTT_CUDA_TRY(cudaGetLastError());
    }
    // a4
    {
      JacArgs ja;
      // per-site block width: the widest WB whose two blocks of this site's (capacity) rows fit
      // in shared memory -- the plan's WB is sized for the tallest site of the sweep
      int WBq = P.WB;
      size_t smq = P.jac_smem;
      int Gq = P.Gjac;
      if (!getenv("QTT_COOP_WB")) {
        WBq = kWarps;
        const long long rows = tq_cand ? n_cap : m_cap;
        while (WBq > 1 && 2 * WBq * (rows + 1) * 8 > 200 * 1024) WBq /= 2;
        WBq = std::max(WBq, P.WB);
        const long long pq = std::min(m_cap, n_cap);
        Gq = (int)std::min<long long>(g_sms, std::max<long long>(1, (pq + 2 * WBq - 1) / (2 * WBq)));
        smq = sizeof(double) * (2 * WBq * rows + 2 * WBq);
      }
      ja.dims = dims_j; ja.A = Bf.A; ja.bar = Bf.bar + 1; ja.flags = Bf.flags; ja.ver = Bf.ver; ja.part = Bf.part; ja.nrm = Bf.s2; ja.G = Gq; ja.WB = WBq;
      ja.noise_ok = noise_ok(io.eps, P.pcap); ja.skip = cqt_ok;
      ja.sweeps_out = io.sweeps ? io.sweeps + q : Bf.sweeps_scratch; ja.status = io.status;
      QTT_CUDA_TRY(cudaMemsetAsync(Bf.flags, 0, sizeof(int) * 3, s));
      QTT_CUDA_TRY(cudaMemsetAsync(Bf.ver, 0, sizeof(int) * (P.pcap + 2), s));
      qtt_status_t st = coop_launch((const void *)k_jacobi_coop, Gq, smq, &ja, s);
      if (st != QTT_OK) return st;
    }
    // a5/a6
    {
      FinishArgs fa;
      fa.dims = dims_j; fa.A = Bf.A; fa.Cq = io.Cq[q]; fa.yr_next = io.yr + q + 1; fa.delta2 = io.delta2 + q;
      fa.sigma = io.sigma ? io.sigma + (size_t)q * io.sigma_stride : nullptr; fa.sigma_stride = io.sigma_stride;
      fa.s2 = Bf.s2; fa.perm = Bf.perm; fa.eps = io.eps; fa.max_rank = io.max_rank; fa.status = io.status;
      fa.carry = Bf.spec + 2; fa.T = Bf.T; fa.Gout = Bf.G; fa.skip = cqt_ok;
      k_finish<<<1, kThreads, 0, s>>>(fa);
      QTT_CUDA_TRY(cudaGetLastError());
      if (cqt_ok) {
        k_cqt_finish<<<1, 32, 0, s>>>(cqt_ok, Bf.dims, io.yr + q + 1, io.delta2 + q, Bf.spec + 2,
                                      io.sweeps ? io.sweeps + q : nullptr);
        QTT_CUDA_TRY(cudaGetLastError());
      }
      if (tq) {                                    // U_T = Q [U_R; 0]
        QapplyArgs qa2;
        qa2.dims = Bf.dims; qa2.dims_j = dims_j; qa2.tq = tq; qa2.Yw = Bf.Tw;
        qa2.tau = (double *)(ws + P.off_tqTau); qa2.C = io.Cq[q];
        qa2.part = Bf.part; qa2.wtot = Bf.wtot; qa2.gram = Bf.gram; qa2.carry = Bf.spec + 2;
        qa2.bar = Bf.bar; qa2.G = tq_G; qa2.RB = tq_RB;
        qtt_status_t st = coop_launch((const void *)k_qapply_coop, tq_G, tq_smem, &qa2, s);
        if (st != QTT_OK) return st;
      }
    }
    launch_gemm_spec(Bf.spec + 2, io.cap[q + 1], n_cap, 1, 1, false, io.tf32, s);
    QTT_CUDA_TRY(cudaGetLastError());
  }
  return QTT_OK;
}

__global__ void k_copy_member(const double *src, double *dst, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

__global__ void k_fill_ranks(int *r, const int *vals, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) r[i] = vals[i];
}

// ------------------------------------------------------------------ host entry

struct OperandPre {       // mirrored-truncate a1 plan for one operand
  int active;
  int L;
  std::vector<int> legs, ranks;          // original (site order)
  std::vector<int> lm, rm, capm;         // mirrored legs, mirrored ranks, truncate-sweep output caps
  std::vector<long long> mel, zel;
  SweepPlan plan;
  size_t off_M, off_Z, off_zr, off_zd, off_zn, off_ws, total;
};

static qtt_status_t plan_operand(int L, const std::vector<int> &legs, const std::vector<int> &ranks, OperandPre &O) {
  O.active = 1; O.L = L; O.legs = legs; O.ranks = ranks;
  O.lm.resize(L); O.rm.resize(L + 1); O.capm.assign(L + 1, 1);
  for (int q = 0; q < L; ++q) O.lm[q] = legs[L - 1 - q];
  for (int q = 0; q <= L; ++q) O.rm[q] = ranks[L - q];
  for (int q = 0; q < L; ++q) {
    long long c = (long long)O.capm[q] * O.lm[q];
    c = std::min<long long>(c, O.rm[q + 1]);
    O.capm[q + 1] = (q == L - 1) ? 1 : (int)c;
  }
  std::vector<int> ones(L + 1, 1);
  qtt_status_t st = plan_sweep(L, O.lm, O.lm, O.rm, ones, O.capm, TRUNCATE, O.plan);
  if (st != QTT_OK) return st;
  O.mel.resize(L); O.zel.resize(L);
  size_t me = 0, ze = 0;
  for (int q = 0; q < L; ++q) {
    O.mel[q] = (long long)O.rm[q] * O.lm[q] * O.rm[q + 1];
    O.zel[q] = (long long)O.capm[q] * O.lm[q] * O.capm[q + 1];
    me += O.mel[q]; ze += O.zel[q];
  }
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  O.off_M = take(8 * me); O.off_Z = take(8 * ze); O.off_zr = take(4 * (L + 1)); O.off_zd = take(8 * (L + 1));
  O.off_zn = take(8); O.off_ws = take(O.plan.total);
  O.total = off;
  return QTT_OK;
}

struct RankRow {
  int v[65];
};
__global__ void k_set_ranks(int *dst, RankRow row, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = row.v[i];
}

// Right-orthonormalise one member's operand in place (slot base + off[q], packed at its
// capacity ranks O.ranks) by the mirrored truncate sweep; writes its device rank row.
static qtt_status_t orth_operand(const OperandPre &O, double *base, const std::vector<long long> &off, int *rank_row,
                                 int *status, char *ws, cudaStream_t s) {
  const int L = O.L;
  double *M = (double *)(ws + O.off_M), *Z = (double *)(ws + O.off_Z);
  int *zr = (int *)(ws + O.off_zr);
  double *zd = (double *)(ws + O.off_zd), *zn = (double *)(ws + O.off_zn);
  std::vector<double *> Mp(L), Zp(L);
  size_t om = 0, oz = 0;
  for (int q = 0; q < L; ++q) { Mp[q] = M + om; om += O.mel[q]; Zp[q] = Z + oz; oz += O.zel[q]; }
  MirrorL a;
  memset(&a, 0, sizeof(a));
  a.L = L; a.pad = 1; a.src_ranks = nullptr;
  for (int q = 0; q < L; ++q) { a.dm[q] = O.legs[q]; a.src[q] = base + off[q]; a.dst[q] = Mp[q]; }
  for (int q = 0; q <= L; ++q) a.cap_src[q] = O.ranks[q];
  k_mirror_l<<<L, kThreads, 0, s>>>(a);
  QTT_CUDA_TRY(cudaGetLastError());
  // the mirrored input is packed at its capacity ranks: constant rank row in the rank_row slot
  RankRow rr;
  for (int q = 0; q <= L; ++q) rr.v[q] = O.rm[q];
  k_set_ranks<<<1, 64, 0, s>>>(rank_row, rr, L + 1);
  QTT_CUDA_TRY(cudaGetLastError());
  SweepIO io;
  io.L = L; io.kind = TRUNCATE; io.d = O.lm; io.dj = O.lm; io.cap = O.capm; io.xcap_r = O.rm;
  io.ocap_r.assign(L + 1, 1);
  io.Xq.assign(Mp.begin(), Mp.end());
  io.Oq.assign(L, nullptr);
  io.xr = rank_row; io.orr = nullptr; io.yr = zr;
  io.Cq.assign(Zp.begin(), Zp.end());
  io.delta2 = zd; io.norm2 = zn; io.sigma = nullptr; io.sigma_stride = 1; io.sweeps = nullptr; io.status = status;
  io.eps = 0.0; io.max_rank = 0;
  qtt_status_t st = run_sweep(io, O.plan, ws + O.off_ws, s);
  if (st != QTT_OK) return st;
  // mirror back (packed at the sweep's ranks) into the operand slot, ranks -> rank_row
  MirrorL b;
  memset(&b, 0, sizeof(b));
  b.L = L; b.pad = 0; b.src_ranks = zr; b.dst_ranks = rank_row;
  for (int q = 0; q < L; ++q) { b.dm[q] = O.lm[q]; b.src[q] = Zp[q]; b.dst[q] = base + off[q]; }
  for (int q = 0; q <= L; ++q) b.cap_src[q] = O.capm[q];
  k_mirror_l<<<L, kThreads, 0, s>>>(b);
  QTT_CUDA_TRY(cudaGetLastError());
  return QTT_OK;
}

struct LargeLayout {
  OperandPre px, po;
  SweepPlan main;
  size_t off_xo, off_xr, off_or, off_oo, off_scratch, total;
};

static qtt_status_t large_layout(const Shape &S, uint32_t flags, LargeLayout &Ly) {
  const int L = S.L;
  std::vector<int> xlegs(L), olegs(L);
  for (int q = 0; q < L; ++q) {
    xlegs[q] = S.dj[q];
    olegs[q] = (S.kind == MATVEC) ? S.d[q] * S.dj[q] : S.d[q];
  }
  qtt_status_t st = plan_operand(L, xlegs, S.xr, Ly.px);
  if (st != QTT_OK) return st;
  Ly.po.active = 0; Ly.po.total = 0;
  if (S.kind != TRUNCATE && !(flags & QTT_NO_OPERATOR_ORTH)) {
    st = plan_operand(L, olegs, S.orr, Ly.po);
    if (st != QTT_OK) return st;
  }
  st = plan_sweep(L, S.d, S.dj, S.xr, S.orr, S.cap, S.kind, Ly.main);
  if (st != QTT_OK) return st;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  Ly.off_xo = take(8 * (size_t)S.xo_elems * S.B);
  Ly.off_oo = take(8 * (size_t)S.oo_elems * (S.shared_op ? 1 : S.B));
  Ly.off_xr = take(4 * (size_t)(S.L + 1) * S.B);
  Ly.off_or = take(4 * (size_t)(S.L + 1) * S.B);
  Ly.off_scratch = take(std::max(std::max(Ly.px.total, Ly.po.total), Ly.main.total));
  Ly.total = off;
  return QTT_OK;
}

size_t large_workspace_bytes(const Shape &S) {
  LargeLayout Ly;
  if (large_layout(S, 0, Ly) != QTT_OK) return 0;
  return Ly.total;
}

qtt_status_t large_zipup(const Shape &S, const qtt_trains_t *op, const qtt_trains_t *x, uint32_t flags,
                         const LargeIO &io, void *workspace, size_t workspace_bytes, cudaStream_t s) {
  LargeLayout Ly;
  qtt_status_t st = large_layout(S, flags, Ly);
  if (st != QTT_OK) return st;
  if (workspace_bytes < Ly.total) { set_error("workspace %zu bytes < required %zu", workspace_bytes, Ly.total); return QTT_ECAPACITY; }
  char *ws = (char *)workspace;
  double *Xo = (double *)(ws + Ly.off_xo), *Oo = (double *)(ws + Ly.off_oo);
  int *xr = (int *)(ws + Ly.off_xr), *orr = (int *)(ws + Ly.off_or);
  char *scratch = ws + Ly.off_scratch;
  const int L = S.L, B = S.B;
  const int nop = (S.kind == TRUNCATE) ? 0 : (S.shared_op ? 1 : B);
  // copy operands into the workspace slots and set the capacity rank rows
  for (int q = 0; q < L; ++q) {
    const long long nx = (long long)S.xr[q] * S.dj[q] * S.xr[q + 1];
    for (int b = 0; b < B; ++b) {
      k_copy_member<<<(unsigned)std::min<long long>((nx + 255) / 256, 4096), 256, 0, s>>>(
          (const double *)x->cores[q] + (size_t)b * nx, Xo + (size_t)b * S.xo_elems + S.xoff[q], nx);
    }
    if (nop) {
      const long long no = S.ooff[q + 1] - S.ooff[q];
      for (int b = 0; b < nop; ++b)
        k_copy_member<<<(unsigned)std::min<long long>((no + 255) / 256, 4096), 256, 0, s>>>(
            (const double *)op->cores[q] + (size_t)b * no, Oo + (size_t)b * S.oo_elems + S.ooff[q], no);
    }
  }
  QTT_CUDA_TRY(cudaGetLastError());
  {
    RankRow rx, ro;
    for (int q = 0; q <= L; ++q) { rx.v[q] = S.xr[q]; ro.v[q] = S.orr[q]; }
    for (int b = 0; b < B; ++b) {
      k_set_ranks<<<1, 64, 0, s>>>(xr + (size_t)b * (L + 1), rx, L + 1);
      k_set_ranks<<<1, 64, 0, s>>>(orr + (size_t)b * (L + 1), ro, L + 1);
    }
    QTT_CUDA_TRY(cudaGetLastError());
  }
  // a1: right-orthonormalise (mirrored truncate sweeps)
  for (int b = 0; b < B; ++b) {
    st = orth_operand(Ly.px, Xo + (size_t)b * S.xo_elems, S.xoff, xr + (size_t)b * (L + 1), io.status, scratch, s);
    if (st != QTT_OK) return st;
  }
  if (Ly.po.active) {
    for (int b = 0; b < nop; ++b) {
      st = orth_operand(Ly.po, Oo + (size_t)b * S.oo_elems, S.ooff, orr + (size_t)b * (L + 1), io.status, scratch, s);
      if (st != QTT_OK) return st;
    }
    if (S.shared_op)
      for (int b = 1; b < B; ++b)
        QTT_CUDA_TRY(cudaMemcpyAsync(orr + (size_t)b * (L + 1), orr, sizeof(int) * (L + 1), cudaMemcpyDeviceToDevice, s));
  }
  // a2..a7 per member
  for (int b = 0; b < B; ++b) {
    SweepIO sw;
    sw.L = L; sw.kind = S.kind; sw.d = S.d; sw.dj = S.dj; sw.cap = S.cap; sw.xcap_r = S.xr; sw.ocap_r = S.orr;
    sw.tf32 = (flags & (1u << 30)) != 0;        // fp32 variant (zipup.cu kFlagTF32)
    sw.Xq.resize(L); sw.Oq.resize(L); sw.Cq.resize(L);
    for (int q = 0; q < L; ++q) {
      sw.Xq[q] = Xo + (size_t)b * S.xo_elems + S.xoff[q];
      sw.Oq[q] = nop ? Oo + (size_t)(S.shared_op ? 0 : b) * S.oo_elems + S.ooff[q] : nullptr;
      sw.Cq[q] = (double *)io.out->cores[q] + (size_t)b * ((long long)io.out->ranks[q] * S.d[q] * io.out->ranks[q + 1]);
    }
    sw.xr = xr + (size_t)b * (L + 1);
    sw.orr = orr + (size_t)b * (L + 1);
    sw.yr = io.out_ranks + (size_t)b * (L + 1);
    sw.delta2 = io.delta2 + (size_t)b * L;
    sw.norm2 = io.norm2 + b;
    sw.sigma = io.sigma ? io.sigma + (size_t)b * (L - 1) * io.sigma_stride : nullptr;
    sw.sigma_stride = io.sigma_stride;
    sw.sweeps = io.sweeps ? io.sweeps + (size_t)b * L : nullptr;
    sw.status = io.status; sw.eps = io.eps; sw.max_rank = io.max_rank;
    st = run_sweep(sw, Ly.main, scratch, s);
    if (st != QTT_OK) return st;
  }
  return QTT_OK;
}


// ======================================================================= f4: sharded zip-up
// One zip-up split across processes (qtt.h qtt_zipup_sharded).  Column
// shards of every site matrix by contiguous balanced ranges of the state bond r_{q+1}; each
// shard's slab is reduced to an m x m factor F_t (F_t^T F_t = T_t T_t^T), the factors of all
// shards are all-gathered and stacked, and the R of the stack is the R of T^H (the TSQR
// identity: T T^T = sum_t T_t T_t^T).  a4-a6 then run on R as in the unsharded sweep; the
// carry U_k^T T is formed per slab and all-gathered ("carry exchange").

__device__ __forceinline__ void shard_range(int n, int S, int t, int &lo, int &hi) {
  lo = (int)(((long long)t * n) / S);
  hi = (int)(((long long)(t + 1) * n) / S);
}

// the state core's r'-slice of shard t into a contiguous slab (r, legs, cnt); xr_s[q] = r,
// xr_s[q+1] = cnt (the slab's rank row for k_plan)
struct SlabArgs {
  const double *Xq;
  const int *xr;
  int q, legs, S, t;
  double *slab;
  int *xr_s;
};
__global__ void k_shard_slab(SlabArgs a) {
  const int r = a.xr[a.q], r2 = a.xr[a.q + 1];
  int lo, hi;
  shard_range(r2, a.S, a.t, lo, hi);
  const int cnt = hi - lo;
  const long long n = (long long)r * a.legs * cnt;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i % cnt);
    const long long rj = i / cnt;
    a.slab[i] = a.Xq[rj * r2 + lo + c];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) { a.xr_s[a.q] = r; a.xr_s[a.q + 1] = cnt; }
}

// F_t (mcap x mcap row-major, zero padded) from the shard's QR (R in A, row-major) or, when
// the slab has fewer columns than rows (direct), from the slab itself: F_t = T_t^T
__global__ void k_shard_factor(const SiteDims *dims, const double *A, const double *T, int mcap, double *F) {
  const SiteDims D = *dims;
  const long long n = (long long)mcap * mcap;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / mcap), c = (int)(i % mcap);
    double v = 0.0;
    if (c < D.m) {
      if (!D.direct) v = (j < D.m && c >= j) ? A[(size_t)j * D.m + c] : 0.0;
      else v = (j < D.n) ? T[(size_t)c * D.n + j] : 0.0;
    }
    F[i] = v;
  }
}

// the stacked factors as a "T" for k_qr_coop: Tw (m x S*mcap) row-major, Tw[c][t*mcap + j] =
// F_t[j][c]; the stack's SiteDims: p = m, never direct, k <= kcap = w' r' (the true columns)
struct StackArgs {
  const SiteDims *dims0;
  const double *recv;
  long long f_elems;
  int S, mcap;
  const int *xr, *orr;
  int q, kind;
  double *Tw;
  SiteDims *dims_st;
};
__global__ void k_shard_stack(StackArgs a) {
  const SiteDims D0 = *a.dims0;
  const int m = D0.m, ns = a.S * a.mcap;
  const long long n = (long long)m * ns;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(i / ns), col = (int)(i % ns), t = col / a.mcap, j = col % a.mcap;
    a.Tw[i] = a.recv[(size_t)t * a.f_elems + (size_t)j * a.mcap + c];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    SiteDims D = D0;
    const int w2 = (a.kind == TRUNCATE) ? 1 : a.orr[a.q + 1];
    D.r2 = a.xr[a.q + 1];
    D.w2 = w2;
    D.n = ns;
    D.direct = 0;
    D.p = m;
    D.k = 0;
    D.kcap = w2 * D.r2;
    *a.dims_st = D;
  }
}

// carry slab spec: send_c[s][kk][w'][c] = sum_i C_q[i][kk] T_s[i][w' cnt + c]  (kk < k, c < cnt)
struct CarrySpecArgs {
  const SiteDims *dims_st, *dims_s;
  const double *Cq, *Ts;
  double *out;
  int slice_cap;
  GemmSpec *spec;
};
__global__ void k_shard_carry_spec(CarrySpecArgs a) {
  if (threadIdx.x != 0) return;
  const SiteDims D = *a.dims_st, Ds = *a.dims_s;
  GemmSpec g{};
  g.M = D.k; g.K = D.m; g.N = Ds.r2; g.nz1 = 1; g.nz2 = Ds.w2;
  g.A = a.Cq; g.sam = 1; g.sak = D.k;
  g.B = a.Ts; g.sbk = Ds.n; g.sbn = 1; g.sb2 = Ds.r2;
  g.C = a.out; g.scm = (long long)Ds.w2 * a.slice_cap; g.scn = 1; g.sc2 = a.slice_cap;
  if (Ds.n == 0 || Ds.r2 == 0) g.M = 0;          // empty slab: nothing to write
  *a.spec = g;
}

// full carry G (k, w', r') from the all-gathered slabs
struct AssembleArgs {
  const SiteDims *dims_st;
  const double *recv;
  long long c_elems;
  int S, slice_cap;
  double *G;
};
__global__ void k_shard_assemble(AssembleArgs a) {
  const SiteDims D = *a.dims_st;
  const int k = D.k, w2 = D.w2, r2 = D.r2;
  const long long n = (long long)k * w2 * r2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int rr = (int)(i % r2);
    const long long kw = i / r2;
    const int ww = (int)(kw % w2), kk = (int)(kw / w2);
    int t = (int)(((long long)rr * a.S) / max(r2, 1));
    int lo, hi;
    shard_range(r2, a.S, t, lo, hi);
    while (rr >= hi) { ++t; shard_range(r2, a.S, t, lo, hi); }
    while (rr < lo) { --t; shard_range(r2, a.S, t, lo, hi); }
    a.G[i] = a.recv[(size_t)t * a.c_elems + ((size_t)kk * w2 + ww) * a.slice_cap + (rr - lo)];
  }
}

struct ShardPlan {
  int S, ls;                        // total shards, local shards
  long long mcap, slab_ncap, slice_cap_max, gcap, xcap, tcap, acap, r_elems, c_elems;
  std::vector<int> slice_cap;       // per site: ceil(xr[q+1] / S)
  int Gqr_s, RB_s, Gqr_st, RB_st, Gjac, WB;
  size_t qr_smem, jac_smem;
  // offsets
  size_t off_xo, off_oo, off_xr, off_or, off_a1, a1_bytes;
  size_t off_G, off_Tst, off_Ast, off_part, off_wtot, off_gram, off_bc, off_s2, off_perm, off_flags, off_ver, off_sw,
      off_bar, off_dims_st, off_spec_st, off_shard, shard_bytes, total;
  // per-shard sub-offsets (relative to off_shard + s * shard_bytes)
  size_t so_slab, so_X, so_T, so_Tw, so_A, so_xr, so_dims, so_spec;
  LargeLayout a1;                   // the unsharded a1 / last-site layout
};

static qtt_status_t plan_shard(const Shape &S_, int world, int ls, uint32_t flags, ShardPlan &P) {
  const Shape &S = S_;
  const int L = S.L;
  P.S = world * ls; P.ls = ls;
  P.mcap = 1; P.slab_ncap = 1; P.gcap = 1; P.xcap = 1; P.tcap = 1; P.acap = 1; P.c_elems = 1;
  P.slice_cap.assign(L + 1, 1);
  long long full_ncap = 1;
  for (int q = 0; q < L; ++q) {
    const long long w = (S.kind == TRUNCATE) ? 1 : S.orr[q], w2 = (S.kind == TRUNCATE) ? 1 : S.orr[q + 1];
    const long long m = (long long)S.cap[q] * S.d[q];
    const long long sc = (S.xr[q + 1] + P.S - 1) / P.S;
    P.slice_cap[q] = (int)sc;
    P.mcap = std::max(P.mcap, m);
    P.slab_ncap = std::max(P.slab_ncap, w2 * sc);
    full_ncap = std::max(full_ncap, w2 * S.xr[q + 1]);
    P.gcap = std::max(P.gcap, (long long)S.cap[q] * w * S.xr[q]);
    P.gcap = std::max(P.gcap, (long long)S.cap[q + 1] * w2 * S.xr[q + 1]);
    const long long legs = (S.kind == MATVEC) ? S.dj[q] : S.d[q];
    P.xcap = std::max(P.xcap, (long long)S.cap[q] * w * legs * std::max(sc, (long long)(q == L - 1 ? S.xr[q + 1] : 1)));
    P.tcap = std::max(P.tcap, m * std::max(w2 * sc, (long long)(q == L - 1 ? w2 * S.xr[q + 1] : 1)));
    P.acap = std::max(P.acap, m * std::min(m, w2 * sc));
    P.c_elems = std::max(P.c_elems, (long long)S.cap[q + 1] * w2 * sc);
  }
  P.acap = std::max(P.acap, P.mcap * P.mcap);
  P.r_elems = P.mcap * P.mcap;
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  auto qr_geom = [&](long long rows, int &Gq, int &RB) -> qtt_status_t {
    Gq = (int)std::min<long long>(g_sms, std::max<long long>(1, (rows + 31) / 32));
    RB = (int)((rows + Gq - 1) / Gq);
    RB = ((RB + 31) / 32) * 32;
    if (RB > kQrRowsMax) { set_error("sharded zip-up: %lld rows of T^H per shard too many", rows); return QTT_EUNSUPPORTED; }
    return QTT_OK;
  };
  qtt_status_t st = qr_geom(P.slab_ncap, P.Gqr_s, P.RB_s);
  if (st != QTT_OK) return st;
  st = qr_geom((long long)P.S * P.mcap, P.Gqr_st, P.RB_st);
  if (st != QTT_OK) return st;
  P.qr_smem = sizeof(double) * ((size_t)kNb * std::max(P.RB_s, P.RB_st) + 32 + kNb * kNb + 2 * kNb + kNb * 64);
  int WB = kWarps;
  while (WB > 1 && 2 * WB * (P.mcap + 1) * 8 > 200 * 1024) WB /= 2;
  if (2 * WB * (P.mcap + 1) * 8 > 200 * 1024) { set_error("sharded zip-up: m = %lld too large", P.mcap); return QTT_EUNSUPPORTED; }
  P.WB = WB;
  P.Gjac = (int)std::min<long long>(g_sms, std::max<long long>(1, (P.mcap + 2 * WB - 1) / (2 * WB)));
  P.jac_smem = sizeof(double) * (2 * WB * P.mcap + 2 * WB);
  st = large_layout(S, flags, P.a1);  // unsharded layout: a1 operand slots + scratch (also the last site)
  if (st != QTT_OK) return st;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  P.off_a1 = take(P.a1.total);
  P.off_G = take(8 * P.gcap);
  P.off_Tst = take(8 * (size_t)P.mcap * P.S * P.mcap);
  P.off_Ast = take(8 * (size_t)P.mcap * P.mcap);
  const int Gmax = std::max(std::max(P.Gqr_s, P.Gqr_st), P.Gjac);
  P.off_part = take(8 * ((size_t)Gmax * kNb * P.mcap + (size_t)Gmax * kNb * kNb + 16));
  P.off_wtot = take(8 * (size_t)kNb * P.mcap);
  P.off_gram = take(8 * kNb * kNb);
  P.off_bc = take(8 * 64);
  P.off_s2 = take(8 * P.mcap);
  P.off_perm = take(4 * P.mcap);
  P.off_flags = take(4 * 4);
  P.off_ver = take(4 * ((size_t)P.mcap + 2));
  P.off_sw = take(4 * 4);
  P.off_bar = take(sizeof(GridBar) * 2);
  P.off_dims_st = take(sizeof(SiteDims));
  P.off_spec_st = take(sizeof(GemmSpec) * 3);
  size_t so = 0;
  auto stake = [&](size_t bytes) { size_t o = so; so += (bytes + 255) & ~size_t(255); return o; };
  long long slab_max = 1;
  for (int q = 0; q < L; ++q) {
    const long long legs = (S.kind == MATVEC) ? S.dj[q] : S.d[q];
    slab_max = std::max(slab_max, (long long)S.xr[q] * legs * P.slice_cap[q]);
  }
  P.so_slab = stake(8 * slab_max);
  P.so_X = stake(8 * P.xcap);
  P.so_T = stake(8 * P.tcap);
  P.so_Tw = stake(8 * P.tcap);
  P.so_A = stake(8 * P.acap);
  P.so_xr = stake(4 * (L + 1));
  P.so_dims = stake(sizeof(SiteDims));
  P.so_spec = stake(sizeof(GemmSpec) * 4);
  P.shard_bytes = so;
  P.off_shard = take(so * ls);
  P.total = off;
  (void)full_ncap;
  return QTT_OK;
}

qtt_status_t sharded_sizes(const Shape &S, int world, int ls, uint32_t flags, size_t *r_elems, size_t *c_elems,
                           size_t *ws_bytes) {
  ShardPlan P;
  qtt_status_t st = plan_shard(S, world, ls, flags, P);
  if (st != QTT_OK) return st;
  if (r_elems) *r_elems = (size_t)P.r_elems;
  if (c_elems) *c_elems = (size_t)P.c_elems;
  if (ws_bytes) *ws_bytes = P.total;
  return QTT_OK;
}

static qtt_status_t shard_exchange(const qtt_shard_comm_t *c, int phase, const ShardPlan &P, cudaStream_t s) {
  if (c->allgather) {
    if (c->allgather(phase, c->user) != 0) { set_error("allgather callback failed (phase %d)", phase); return QTT_EINVAL; }
    return QTT_OK;
  }
  const size_t n = (phase == 0) ? (size_t)P.r_elems : (size_t)P.c_elems;
  const double *src = (phase == 0) ? c->send_r : c->send_c;
  double *dst = (phase == 0) ? c->recv_r : c->recv_c;
  QTT_CUDA_TRY(cudaMemcpyAsync(dst + (size_t)c->rank * P.ls * n, src, sizeof(double) * n * P.ls,
                               cudaMemcpyDeviceToDevice, s));
  return QTT_OK;
}

qtt_status_t large_zipup_sharded(const Shape &S, const qtt_trains_t *op, const qtt_trains_t *x, uint32_t flags,
                                 const LargeIO &io, const qtt_shard_comm_t *comm, void *workspace,
                                 size_t workspace_bytes, cudaStream_t s) {
  ShardPlan P;
  qtt_status_t st = plan_shard(S, comm->world, comm->local_shards, flags, P);
  if (st != QTT_OK) return st;
  if (!workspace || workspace_bytes < P.total) {
    set_error("workspace %zu bytes < required %zu", workspace_bytes, P.total);
    return QTT_ECAPACITY;
  }
  const int L = S.L, kind = S.kind;
  char *ws = (char *)workspace;
  // ---- a1 on the full operands (every process, identical results): the unsharded layout
  char *wa = ws + P.off_a1;
  double *Xo = (double *)(wa + P.a1.off_xo), *Oo = (double *)(wa + P.a1.off_oo);
  int *xr = (int *)(wa + P.a1.off_xr), *orr = (int *)(wa + P.a1.off_or);
  char *scratch = wa + P.a1.off_scratch;
  const bool has_op = kind != TRUNCATE;
  for (int q = 0; q < L; ++q) {
    const long long nx = (long long)S.xr[q] * S.dj[q] * S.xr[q + 1];
    k_copy_member<<<(unsigned)std::min<long long>((nx + 255) / 256, 4096), 256, 0, s>>>(
        (const double *)x->cores[q], Xo + S.xoff[q], nx);
    if (has_op) {
      const long long no = S.ooff[q + 1] - S.ooff[q];
      k_copy_member<<<(unsigned)std::min<long long>((no + 255) / 256, 4096), 256, 0, s>>>(
          (const double *)op->cores[q], Oo + S.ooff[q], no);
    }
  }
  QTT_CUDA_TRY(cudaGetLastError());
  {
    RankRow rx, ro;
    for (int q = 0; q <= L; ++q) { rx.v[q] = S.xr[q]; ro.v[q] = S.orr[q]; }
    k_set_ranks<<<1, 64, 0, s>>>(xr, rx, L + 1);
    k_set_ranks<<<1, 64, 0, s>>>(orr, ro, L + 1);
    QTT_CUDA_TRY(cudaGetLastError());
  }
  st = orth_operand(P.a1.px, Xo, S.xoff, xr, io.status, scratch, s);
  if (st != QTT_OK) return st;
  if (P.a1.po.active) {
    st = orth_operand(P.a1.po, Oo, S.ooff, orr, io.status, scratch, s);
    if (st != QTT_OK) return st;
  }
  QTT_CUDA_TRY(cudaFuncSetAttribute(k_qr_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  QTT_CUDA_TRY(cudaFuncSetAttribute(k_jacobi_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  QTT_CUDA_TRY(cudaFuncSetAttribute(k_gemm_dmma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)dgemm::SMEM_BYTES));
  QTT_CUDA_TRY(cudaFuncSetAttribute(k_gemm_dmma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)dgemm::SMEM_BYTES));
  // ---- shared buffers
  double *G = (double *)(ws + P.off_G), *Tst = (double *)(ws + P.off_Tst), *Ast = (double *)(ws + P.off_Ast);
  double *part = (double *)(ws + P.off_part), *wtot = (double *)(ws + P.off_wtot), *gram = (double *)(ws + P.off_gram);
  double *bc = (double *)(ws + P.off_bc), *s2 = (double *)(ws + P.off_s2);
  int *perm = (int *)(ws + P.off_perm), *jflags = (int *)(ws + P.off_flags), *ver = (int *)(ws + P.off_ver);
  int *sw_scr = (int *)(ws + P.off_sw);
  GridBar *bar = (GridBar *)(ws + P.off_bar);
  SiteDims *dims_st = (SiteDims *)(ws + P.off_dims_st);
  GemmSpec *spec_st = (GemmSpec *)(ws + P.off_spec_st);
  QTT_CUDA_TRY(cudaMemsetAsync(bar, 0, sizeof(GridBar) * 2, s));
  k_site0_init<<<1, 32, 0, s>>>(G, io.out_ranks);
  QTT_CUDA_TRY(cudaGetLastError());
  auto shard_base = [&](int sl) { return ws + P.off_shard + (size_t)sl * P.shard_bytes; };
  const int grank = comm->rank;
  for (int q = 0; q < L; ++q) {
    const long long w = (kind == TRUNCATE) ? 1 : S.orr[q], w2 = (kind == TRUNCATE) ? 1 : S.orr[q + 1];
    const long long legs = (kind == MATVEC) ? S.dj[q] : S.d[q];
    const long long m_cap = (long long)S.cap[q] * S.d[q];
    const double *Xq = Xo + S.xoff[q];
    const double *Oq = has_op ? Oo + S.ooff[q] : nullptr;
    double *Cq = (double *)io.out->cores[q];
    auto contract = [&](char *sb, const double *xsrc, const int *xr_row, long long ncols_cap) -> qtt_status_t {
      SiteDims *dims = (SiteDims *)(sb + P.so_dims);
      GemmSpec *spec = (GemmSpec *)(sb + P.so_spec);
      double *X = (double *)(sb + P.so_X), *T = (double *)(sb + P.so_T);
      PlanArgs pa;
      pa.q = q; pa.L = L; pa.kind = kind; pa.d = S.d[q]; pa.dj = S.dj[q];
      pa.xr = xr_row; pa.orr = orr; pa.yr = io.out_ranks;
      pa.Xq = xsrc; pa.Oq = Oq;
      pa.G = G; pa.X = X; pa.T = T; pa.Cq = Cq;
      pa.dims = dims; pa.spec = spec;
      k_plan<<<1, 32, 0, s>>>(pa);
      QTT_CUDA_TRY(cudaGetLastError());
      launch_gemm_spec(spec + 0, (long long)S.cap[q] * w, legs * ncols_cap, 1, 1, true, false, s);
      QTT_CUDA_TRY(cudaGetLastError());
      const unsigned ew = (unsigned)std::min<long long>((m_cap * w2 * ncols_cap + kThreads - 1) / kThreads, 8192);
      if (kind == MATVEC) {
        k_mpo_apply<<<std::max(ew, 1u), kThreads, 0, s>>>(dims, X, Oq, T);
        QTT_CUDA_TRY(cudaGetLastError());
      } else if (kind == HADAMARD) {
        launch_gemm_spec(spec + 1, w2, ncols_cap, S.cap[q], S.d[q], false, false, s);
        QTT_CUDA_TRY(cudaGetLastError());
      }
      return QTT_OK;
    };
    if (q == L - 1) {            // a7: unsharded on every process
      char *sb = shard_base(0);
      st = contract(sb, Xq, xr, S.xr[q + 1]);
      if (st != QTT_OK) return st;
      k_last<<<1, kThreads, 0, s>>>((SiteDims *)(sb + P.so_dims), (double *)(sb + P.so_T), Cq, io.norm2,
                                    io.delta2 + q, io.out_ranks + L, io.status);
      QTT_CUDA_TRY(cudaGetLastError());
      if (io.sweeps) QTT_CUDA_TRY(cudaMemsetAsync(io.sweeps + q, 0, sizeof(int), s));
      break;
    }
    const int sc = P.slice_cap[q];
    // 1. local shards: slab, contraction, factor F_t
    for (int sl = 0; sl < P.ls; ++sl) {
      char *sb = shard_base(sl);
      const int t = grank * P.ls + sl;
      SlabArgs ka{Xq, xr, q, (int)legs, P.S, t, (double *)(sb + P.so_slab), (int *)(sb + P.so_xr)};
      const long long nslab = (long long)S.xr[q] * legs * sc;
      k_shard_slab<<<(unsigned)std::max<long long>(1, std::min<long long>((nslab + 255) / 256, 4096)), 256, 0, s>>>(ka);
      QTT_CUDA_TRY(cudaGetLastError());
      st = contract(sb, (double *)(sb + P.so_slab), (int *)(sb + P.so_xr), sc);
      if (st != QTT_OK) return st;
      SiteDims *dims = (SiteDims *)(sb + P.so_dims);
      double *T = (double *)(sb + P.so_T), *Tw = (double *)(sb + P.so_Tw), *A = (double *)(sb + P.so_A);
      const unsigned ew = (unsigned)std::max<long long>(1, std::min<long long>((m_cap * w2 * sc + kThreads - 1) / kThreads, 8192));
      k_copy_T<<<ew, kThreads, 0, s>>>(dims, T, Tw, A);
      QTT_CUDA_TRY(cudaGetLastError());
      QrArgs qa;
      qa.dims = dims; qa.Tw = Tw; qa.Rout = A; qa.part = part; qa.wtot = wtot; qa.gram = gram;
      qa.bc = bc; qa.bar = bar; qa.G = P.Gqr_s; qa.RB = P.RB_s; qa.mcap = (int)P.mcap; qa.skip = nullptr; qa.tau_out = nullptr;
      st = coop_launch((const void *)k_qr_coop, P.Gqr_s, P.qr_smem, &qa, s);
      if (st != QTT_OK) return st;
      const long long fe = P.r_elems;
      k_shard_factor<<<(unsigned)std::min<long long>((fe + 255) / 256, 4096), 256, 0, s>>>(
          dims, A, T, (int)P.mcap, comm->send_r + (size_t)sl * fe);
      QTT_CUDA_TRY(cudaGetLastError());
    }
    // 2. exchange the factors
    st = shard_exchange(comm, 0, P, s);
    if (st != QTT_OK) return st;
    // 3. R of the stack, Jacobi, truncation + emit
    {
      StackArgs sa{(SiteDims *)(shard_base(0) + P.so_dims), comm->recv_r, P.r_elems, P.S, (int)P.mcap, xr, orr,
                   q, kind, Tst, dims_st};
      if (kind == TRUNCATE) sa.orr = xr;          // unused (w2 = 1)
      const long long ne = m_cap * P.S * P.mcap;
      k_shard_stack<<<(unsigned)std::min<long long>((ne + 255) / 256, 8192), 256, 0, s>>>(sa);
      QTT_CUDA_TRY(cudaGetLastError());
      QrArgs qa;
      qa.dims = dims_st; qa.Tw = Tst; qa.Rout = Ast; qa.part = part; qa.wtot = wtot; qa.gram = gram;
      qa.bc = bc; qa.bar = bar; qa.G = P.Gqr_st; qa.RB = P.RB_st; qa.mcap = (int)P.mcap; qa.skip = nullptr; qa.tau_out = nullptr;
      st = coop_launch((const void *)k_qr_coop, P.Gqr_st, P.qr_smem, &qa, s);
      if (st != QTT_OK) return st;
      JacArgs ja;
      ja.dims = dims_st; ja.A = Ast; ja.bar = bar + 1; ja.flags = jflags; ja.ver = ver; ja.part = part; ja.nrm = s2;
      ja.G = P.Gjac; ja.WB = P.WB;
      ja.noise_ok = noise_ok(io.eps, (int)P.mcap); ja.skip = nullptr;
      ja.sweeps_out = io.sweeps ? io.sweeps + q : sw_scr; ja.status = io.status;
      QTT_CUDA_TRY(cudaMemsetAsync(jflags, 0, sizeof(int) * 3, s));
      QTT_CUDA_TRY(cudaMemsetAsync(ver, 0, sizeof(int) * (P.mcap + 2), s));
      st = coop_launch((const void *)k_jacobi_coop, P.Gjac, P.jac_smem, &ja, s);
      if (st != QTT_OK) return st;
      FinishArgs fa;
      fa.dims = dims_st; fa.A = Ast; fa.Cq = Cq; fa.yr_next = io.out_ranks + q + 1; fa.delta2 = io.delta2 + q;
      fa.sigma = io.sigma ? io.sigma + (size_t)q * io.sigma_stride : nullptr; fa.sigma_stride = io.sigma_stride;
      fa.s2 = s2; fa.perm = perm; fa.eps = io.eps; fa.max_rank = io.max_rank; fa.status = io.status;
      fa.carry = spec_st + 2; fa.T = Tst; fa.Gout = G; fa.skip = nullptr;
      k_finish<<<1, kThreads, 0, s>>>(fa);
      QTT_CUDA_TRY(cudaGetLastError());
    }
    // 4. carry slabs U_k^T T_t
    for (int sl = 0; sl < P.ls; ++sl) {
      char *sb = shard_base(sl);
      GemmSpec *cs = (GemmSpec *)(sb + P.so_spec) + 3;
      CarrySpecArgs ca{dims_st, (SiteDims *)(sb + P.so_dims), Cq, (double *)(sb + P.so_T),
                       comm->send_c + (size_t)sl * P.c_elems, sc, cs};
      k_shard_carry_spec<<<1, 32, 0, s>>>(ca);
      QTT_CUDA_TRY(cudaGetLastError());
      launch_gemm_spec(cs, S.cap[q + 1], sc, 1, w2, false, false, s);
      QTT_CUDA_TRY(cudaGetLastError());
    }
    // 5. exchange the carry slabs, assemble the full carry
    st = shard_exchange(comm, 1, P, s);
    if (st != QTT_OK) return st;
    {
      AssembleArgs aa{dims_st, comm->recv_c, P.c_elems, P.S, sc, G};
      const long long ne = (long long)S.cap[q + 1] * w2 * S.xr[q + 1];
      k_shard_assemble<<<(unsigned)std::max<long long>(1, std::min<long long>((ne + 255) / 256, 8192)), 256, 0, s>>>(aa);
      QTT_CUDA_TRY(cudaGetLastError());
    }
  }
  return QTT_OK;
}

}  // namespace qtt


using namespace qtt;

static qtt_status_t sharded_check(const char *subs, const qtt_trains_t *op, const qtt_trains_t *x, int32_t max_rank,
                                  int32_t world, int32_t ls, Shape &S) {
  if (!x || x->dtype != QTT_F64 || (op && op->dtype != QTT_F64)) {
    set_error("qtt_zipup_sharded: QTT_F64 trains only");
    return QTT_EUNSUPPORTED;
  }
  qtt_status_t st = qtt_zipup_analyse(subs, op, x, max_rank, S);
  if (st != QTT_OK) return st;
  if (S.B != 1) { set_error("qtt_zipup_sharded: batch must be 1 (one zip-up split across processes)"); return QTT_EUNSUPPORTED; }
  if (world < 1 || ls < 1) { set_error("qtt_zipup_sharded: world %d / local_shards %d", world, ls); return QTT_EINVAL; }
  return QTT_OK;
}

extern "C" {

qtt_status_t qtt_zipup_sharded_sizes(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                     int32_t max_rank, int32_t world, int32_t local_shards, size_t *r_elems,
                                     size_t *c_elems, size_t *workspace_bytes) {
  Shape S;
  qtt_status_t st = sharded_check(subscripts, op, x, max_rank, world, local_shards, S);
  if (st != QTT_OK) return st;
  return sharded_sizes(S, world, local_shards, 0, r_elems, c_elems, workspace_bytes);
}

qtt_status_t qtt_zipup_sharded(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x, double eps,
                               int32_t max_rank, uint32_t flags, const qtt_trains_t *out, int32_t *out_ranks,
                               double *delta2, double *norm2, int32_t *status, double *sigma, int32_t sigma_stride,
                               const qtt_shard_comm_t *comm, void *workspace, size_t workspace_bytes,
                               void *stream) {
  if (!(eps >= 0.0 && eps < 1.0)) { set_error("eps %g outside [0,1)", eps); return QTT_EINVAL; }
  if (flags & QTT_WINDOW2) { set_error("qtt_zipup_sharded: window 1 only"); return QTT_EUNSUPPORTED; }
  if (!comm) { set_error("comm is NULL"); return QTT_EINVAL; }
  Shape S;
  qtt_status_t st = sharded_check(subscripts, op, x, max_rank, comm->world, comm->local_shards, S);
  if (st != QTT_OK) return st;
  if (comm->rank < 0 || comm->rank >= comm->world) { set_error("rank %d outside [0, %d)", comm->rank, comm->world); return QTT_EINVAL; }
  if (comm->world > 1 && !comm->allgather) { set_error("world > 1 needs an allgather callback"); return QTT_EINVAL; }
  if (!comm->send_r || !comm->recv_r || !comm->send_c || !comm->recv_c) { set_error("NULL exchange buffer"); return QTT_EINVAL; }
  if (!out || !out->cores || !out->ranks || !out_ranks || !delta2 || !norm2 || !status) {
    set_error("NULL output argument");
    return QTT_EINVAL;
  }
  if (out->n_sites != S.L || out->batch != 1 || out->n_legs != 1) { set_error("output train shape mismatch"); return QTT_ESHAPE; }
  for (int q = 0; q <= S.L; ++q)
    if (out->ranks[q] < S.cap[q]) {
      set_error("output capacity %d at bond %d below required %d", out->ranks[q], q, S.cap[q]);
      return QTT_ECAPACITY;
    }
  if (sigma && sigma_stride < 1) { set_error("sigma_stride < 1"); return QTT_EINVAL; }
  cudaStream_t s = (cudaStream_t)stream;
  QTT_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), s));
  LargeIO io{out, out_ranks, delta2, norm2, sigma, sigma_stride, nullptr, status, eps, max_rank};
  return large_zipup_sharded(S, op, x, flags, io, comm, workspace, workspace_bytes, s);
}

}  // extern "C"
