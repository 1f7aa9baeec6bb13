// complex.cu -- complex128 zip-up (the tensorized Fourier transform
// of PAPER.md:533-566 is a chain of Hadamard zip-ups of complex trains).
//
// Same steps as the fp64 path (qtt.h qtt_zipup) in complex
// arithmetic, one CTA (256 threads) per member running every step for that member:
//   a1  right-orthonormalise each operand: for q = L-1..1, Householder QR of M^T
//       (M = core q unfolded (r, legs r')), core q <- Q^T, core q-1 <- core q-1 R^T
//       (Q^T has orthonormal rows in the complex sense)
//   a2  T[(c,i),(w',r')] = sum G[c,w,r] x[r,j,r'] op[w,i,j,w']  (Eq. einsum)
//   a3  Householder QR of T^H when m <= n (A = R^H), else A = T
//   a4  one-sided complex Jacobi on the columns of A: pair (i, j) with a = |a_i|^2,
//       b = |a_j|^2, g = a_i^H a_j = |g| e^{i phi}; zeta = (b - a) / (2|g|),
//       t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)), c = 1/sqrt(1+t^2), s = c t (evaluated
//       division-free with two MUFU-seeded rsqrt, as the fp64 path);
//       a_i <- c a_i - s e^{-i phi} a_j,  a_j <- s e^{i phi} a_i + c a_j
//       (the real rotation of the 2x2 Gram matrix after removing the phase of g);
//       sweeps until no pair has |g|^2 > tol^2 a b (tol = m eps); noise-level columns as c-A31
//   a5  truncation rule of SPEC.md:299 (tail sums smallest first), delta2
//   a6  C_q = U[:, :k] (chi, d, k), carry G <- U_k^H T
//   a7  last site C_{L-1} = T, norm2 = ||T||_F^2.
// The member's operands, carry and site matrices live in its slice of the workspace (global
// memory, L1/L2 resident at the Fourier chain's sizes: rank <= 64, d <= 8).  This is the
// complex row's first, plain version: no tensor cores, no register blocking.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "jacobi.cuh"
#include "qr_small.cuh"
#include "large.cuh"

namespace qtt {

namespace cplx {

struct __align__(16) Z {
  double x, y;
};
__device__ __forceinline__ Z mk(double a, double b) { return Z{a, b}; }
__device__ __forceinline__ Z add(Z a, Z b) { return Z{a.x + b.x, a.y + b.y}; }
__device__ __forceinline__ Z sub(Z a, Z b) { return Z{a.x - b.x, a.y - b.y}; }
__device__ __forceinline__ Z mul(Z a, Z b) { return Z{a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x}; }
__device__ __forceinline__ Z conj(Z a) { return Z{a.x, -a.y}; }
__device__ __forceinline__ Z scl(double s, Z a) { return Z{s * a.x, s * a.y}; }
__device__ __forceinline__ double abs2(Z a) { return a.x * a.x + a.y * a.y; }
// acc += conj(a) * b
__device__ __forceinline__ Z cfma(Z a, Z b, Z acc) {
  return Z{fma(a.x, b.x, fma(a.y, b.y, acc.x)), fma(a.x, b.y, fma(-a.y, b.x, acc.y))};
}
// acc += a * b
__device__ __forceinline__ Z zfma(Z a, Z b, Z acc) {
  return Z{fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y))};
}
__device__ __forceinline__ Z warp_zsum(Z v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// the same operations on a real double: the kernel below is instantiated for both
__device__ __forceinline__ double add(double a, double b) { return a + b; }
__device__ __forceinline__ double sub(double a, double b) { return a - b; }
__device__ __forceinline__ double mul(double a, double b) { return a * b; }
__device__ __forceinline__ double conj(double a) { return a; }
__device__ __forceinline__ double scl(double s, double a) { return s * a; }
__device__ __forceinline__ double abs2(double a) { return a * a; }
__device__ __forceinline__ double cfma(double a, double b, double acc) { return fma(a, b, acc); }
__device__ __forceinline__ double zfma(double a, double b, double acc) { return fma(a, b, acc); }
__device__ __forceinline__ double warp_zsum(double v) { return warp_sum(v); }
__device__ __forceinline__ double re(double a) { return a; }
__device__ __forceinline__ double im(double) { return 0.0; }
__device__ __forceinline__ double re(Z a) { return a.x; }
__device__ __forceinline__ double im(Z a) { return a.y; }
__device__ __forceinline__ bool nz(double a) { return a != 0.0; }
__device__ __forceinline__ bool nz(Z a) { return a.x != 0.0 || a.y != 0.0; }
template <typename S> __device__ __forceinline__ S mk(double r, double i);
template <> __device__ __forceinline__ double mk<double>(double r, double) { return r; }
template <> __device__ __forceinline__ Z mk<Z>(double r, double i) { return Z{r, i}; }
// v + (v of lane ^ o) within `mask`
__device__ __forceinline__ double shx(double v, unsigned mask, int o) { return v + __shfl_xor_sync(mask, v, o); }
__device__ __forceinline__ Z shx(Z v, unsigned mask, int o) {
  return Z{v.x + __shfl_xor_sync(mask, v.x, o), v.y + __shfl_xor_sync(mask, v.y, o)};
}

constexpr int kMaxSweeps = 60;

struct Args {
  int L, B, kind, op_batch;
  int d[64], dj[64], xr0[65], or0[65], cap[65];
  long long xoff[65], ooff[65];        // per-member element offsets of the compact operand copies
  const void *xsrc[64];
  const void *osrc[64];
  void *Cq[64];
  long long Cq_bs[64];
  long long x_bs[64], o_bs[64];        // member stride of the input cores (elements)
  void *ws;                            // per-member scratch (scalars of the instantiated type)
  long long ws_member;                 // scalars per member
  long long xo_n, oo_n, g_n, t_n;      // sizes of the member's regions
  char *iws;                           // per-member int/double scratch
  long long iws_member;                // bytes per member
  int pmax;
  int *yr;                             // out_ranks [B][L+1]
  double *delta2, *norm2, *sigma;
  int sigma_stride;
  int *sweeps, *status;
  double eps;
  int max_rank, orth_op;
  int smem;                            // 1: G, T, H, Q/A, tau in dynamic shared memory
  long long *cycles;                   // optional [B][L][4]: a2, a3, a4, a5-a6 clocks (a1 in [q=0][3])
  int window;                          // 1, or 2 (f4)
  int jreg;                            // real: register-blocked Jacobi (jacobi.cuh) in smem at jsm_off
  long long jsm_off;                   // byte offset of that region in dynamic shared memory
  const int *xr_pre, *orr_pre;         // real: a1 done by k_orth into the member slots ([B][L+1] ranks)
};

// In-place Householder QR of the column-major rows x cols matrix H (ld = rows), K =
// min(rows, cols) reflectors (LAPACK zgeqr2 conventions: H_j = I - tau_j v_j v_j^H,
// v_j[j] = 1, beta real on the diagonal; H_j^H applied to the trailing columns).
template <typename S>
__device__ void house_qr(S *H, int rows, int cols, S *tau, double *red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int K = min(rows, cols);
  __shared__ S s_scal;
  for (int j = 0; j < K; ++j) {
    S *v = H + (size_t)j * rows;
    if (warp == 0) {                    // reflector: warp 0 alone (norm by butterfly)
      double xn = 0.0;
      for (int i = j + 1 + lane; i < rows; i += 32) xn += abs2(v[i]);
      xn = warp_sum(xn);
      if (lane == 0) {
      const S alpha = v[j];
      S t = mk<S>(0.0, 0.0);
      S inv = mk<S>(0.0, 0.0);
      if (xn == 0.0 && im(alpha) == 0.0) {
        t = mk<S>(0.0, 0.0);
      } else {
        const double beta = -copysign(sqrt(abs2(alpha) + xn), re(alpha));
        t = mk<S>((beta - re(alpha)) / beta, -im(alpha) / beta);
        const double dr = re(alpha) - beta, di = im(alpha);   // 1 / (alpha - beta)
        const double dd = dr * dr + di * di;
        inv = mk<S>(dr / dd, -di / dd);
        v[j] = mk<S>(beta, 0.0);
      }
      tau[j] = t;
      s_scal = inv;
      }
      __syncwarp();
      const S inv = s_scal;
      const S t = tau[j];
      if (nz(t))
        for (int i = j + 1 + lane; i < rows; i += 32) v[i] = mul(v[i], inv);
    }
    __syncthreads();
    const S t = tau[j];
    // trailing columns: c <- c - conj(tau) v (v^H c), one warp per column
    if (nz(t)) {
      const S ct = conj(t);
      for (int c = j + 1 + warp; c < cols; c += kWarps) {
        S *col = H + (size_t)c * rows;
        S w = mk<S>(0.0, 0.0);
        for (int i = j + lane; i < rows; i += 32) {
          const S vi = (i == j) ? mk<S>(1.0, 0.0) : v[i];
          w = cfma(vi, col[i], w);
        }
        w = warp_zsum(w);
        const S f = mul(ct, w);
        for (int i = j + lane; i < rows; i += 32) {
          const S vi = (i == j) ? mk<S>(1.0, 0.0) : v[i];
          col[i] = sub(col[i], mul(f, vi));
        }
      }
    }
    __syncthreads();
  }
}

// Q (rows x K, column-major, ld = rows) = H_0 H_1 ... H_{K-1} applied to the first K columns
// of the identity (LAPACK zung2r), from the reflectors left in H by house_qr.
template <typename S>
__device__ void form_q(const S *H, int rows, int K, const S *tau, S *Q) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < rows * K; idx += kThreads) {
    const int i = idx % rows, c = idx / rows;
    Q[idx] = mk<S>((i == c) ? 1.0 : 0.0, 0.0);
  }
  __syncthreads();
  for (int j = K - 1; j >= 0; --j) {
    const S t = tau[j];
    if (!nz(t)) continue;
    const S *v = H + (size_t)j * rows;
    for (int c = j + warp; c < K; c += kWarps) {
      S *col = Q + (size_t)c * rows;
      S w = mk<S>(0.0, 0.0);
      for (int i = j + lane; i < rows; i += 32) {
        const S vi = (i == j) ? mk<S>(1.0, 0.0) : v[i];
        w = cfma(vi, col[i], w);
      }
      w = warp_zsum(w);
      const S f = mul(t, w);
      for (int i = j + lane; i < rows; i += 32) {
        const S vi = (i == j) ? mk<S>(1.0, 0.0) : v[i];
        col[i] = sub(col[i], mul(f, vi));
      }
    }
    __syncthreads();
  }
}

// One-sided Jacobi on the columns of A (rows x p, column-major, ld = rows).  Returns sweeps.
template <typename S>
__device__ int jacobi(S *A, int rows, int p, double noise_eps, double *red) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, hl = lane & 15;
  const unsigned hmask = 0xffffu << (16 * half);
  const double tol = (double)max(rows, 1) * DBL_EPSILON;
  __shared__ int s_rot, s_big, s_fail;
  double tot = 0.0;
  for (int i = tid; i < rows * p; i += kThreads) tot += abs2(A[i]);
  tot = block_sum(tot, red);
  // exact power-of-two scaling to ||A||_F^2 in [1, 4), undone at the end (reading c-A33):
  // keeps |g|^2 and a b of the rotation test clear of under/overflow for any input magnitude
  double scale = 1.0;
  if (tot > 0.0 && isfinite(tot)) {
    const int e = -(ilogb(tot) >> 1);
    if (e != 0) {
      scale = ldexp(1.0, e);
      tot = ldexp(tot, 2 * e);
      for (int i = tid; i < rows * p; i += kThreads) A[i] = scl(scale, A[i]);
      __syncthreads();
    }
  }
  const double noise = noise_eps * tot;
  const int n = p + (p & 1);
  int sweep = 0;
  for (; sweep < kMaxSweeps; ++sweep) {
    if (tid == 0) { s_rot = 0; s_big = 0; }
    __syncthreads();
    int rot = 0, big = 0;
    for (int r = 0; r < n - 1; ++r) {
      // one pair per half-warp (16 lanes): 16 pairs of a round in flight across the 8 warps
      for (int pr = 2 * warp + half; pr < n / 2; pr += 2 * kWarps) {
        // circle method: position 0 fixed, the others rotate
        const int k1 = pr, k2 = n - 1 - pr;
        const int ci = (k1 == 0) ? 0 : 1 + (k1 - 1 + r) % (n - 1);
        const int cj = 1 + (k2 - 1 + r) % (n - 1);
        if (ci >= p || cj >= p) continue;
        S *ai = A + (size_t)ci * rows, *aj = A + (size_t)cj * rows;
        double al = 0.0, be = 0.0;
        S g = mk<S>(0.0, 0.0);
        double al2 = 0.0, be2 = 0.0;
        S g2 = mk<S>(0.0, 0.0);
        int i = hl;
        for (; i + 16 < rows; i += 32) {                // two independent chains
          const S x = ai[i], y = aj[i], x1 = ai[i + 16], y1 = aj[i + 16];
          al += abs2(x); al2 += abs2(x1);
          be += abs2(y); be2 += abs2(y1);
          g = cfma(x, y, g); g2 = cfma(x1, y1, g2);
        }
        al += al2; be += be2; g = add(g, g2);
        for (; i < rows; i += 16) {
          const S x = ai[i], y = aj[i];
          al += abs2(x);
          be += abs2(y);
          g = cfma(x, y, g);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {            // four independent butterflies interleave
          al = shx(al, hmask, o);
          be = shx(be, hmask, o);
          g = shx(g, hmask, o);
        }
        const double ag2 = abs2(g);
        if (al > noise && be > noise && ag2 >= 1e-12 * (al * be)) big = 1;
        if (al > noise && be > noise && ag2 > tol * tol * al * be) {
          // division-free (as the fp64 path): with d = b - a, y = 1/sqrt(d^2 + 4|g|^2),
          // c^2 = (1 + |d| y)/2, z = 1/c: c = c^2 z and s e^{i phi} = sign(d) y z g
          double d = be - al, x2 = fma(d, d, 4.0 * ag2);
          S gg = g;
          if (x2 < 1e-280) {             // keep the MUFU rsqrt seed out of the subnormal range
            const double sc = 1.0 / fmax(fabs(d), sqrt(ag2));
            d *= sc; gg = scl(sc, g);
            x2 = fma(d, d, 4.0 * abs2(gg));
          }
          const double y = fast_rsqrt(x2);
          const double c2 = fma(0.5 * fabs(d), y, 0.5);
          const double z = fast_rsqrt(c2);
          const double c = c2 * z, f = copysign(1.0, d) * y * z;
          const S sp = scl(f, gg), sm = scl(f, conj(gg));
#pragma unroll 4
          for (int i = hl; i < rows; i += 16) {
            const S x = ai[i], y = aj[i];
            ai[i] = sub(scl(c, x), mul(sm, y));
            aj[i] = add(mul(sp, x), scl(c, y));
          }
          rot = 1;
        }
      }
      __syncthreads();
    }
    if (rot) s_rot = 1;
    if (big) s_big = 1;
    __syncthreads();
    const int any = s_rot, anybig = s_big;
    __syncthreads();
    if (!any) { ++sweep; break; }
    // every pair of this sweep started within |cos| < 1e-6: by the quadratic convergence of
    // cyclic Jacobi the next sweep is almost always the verification sweep that rotates nothing
    // -- check that on all pairs at once (no rounds, one barrier) with the sweep's own test
    if (!anybig) {
      if (tid == 0) s_fail = 0;
      __syncthreads();
      int fail = 0;
      for (int e = 2 * warp + half; e < p * p; e += 2 * kWarps) {
        const int ci = e / p, cj = e % p;
        if (cj <= ci) continue;
        const S *ai = A + (size_t)ci * rows, *aj = A + (size_t)cj * rows;
        double al = 0.0, be = 0.0;
        S g = mk<S>(0.0, 0.0);
        for (int i = hl; i < rows; i += 16) {
          const S x = ai[i], y = aj[i];
          al += abs2(x);
          be += abs2(y);
          g = cfma(x, y, g);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
          al = shx(al, hmask, o);
          be = shx(be, hmask, o);
          g = shx(g, hmask, o);
        }
        if (al > noise && be > noise && abs2(g) > tol * tol * al * be) fail = 1;
      }
      if (fail) s_fail = 1;
      __syncthreads();
      const int f = s_fail;
      __syncthreads();
      if (!f) { ++sweep; break; }
    }
  }
  if (scale != 1.0) {
    const double inv = 1.0 / scale;
    for (int i = tid; i < rows * p; i += kThreads) A[i] = scl(inv, A[i]);
    __syncthreads();
  }
  return sweep;
}

// a1 for one operand of member b: copy its cores into the compact slots `dst` (offsets off[q])
// and right-orthonormalise in place; rk[0..L] receives the ranks.
template <typename S>
__device__ void orth_operand(const Args &a, const void *const *src, const long long *sbs, int member, const int *legs,
                             const int *r0, const long long *off, S *dst, int *rk, bool orth, S *H, S *Q, S *tau,
                             double *red) {
  const int tid = threadIdx.x;
  const int L = a.L;
  for (int q = 0; q < L; ++q) {
    const long long n = (long long)r0[q] * legs[q] * r0[q + 1];
    const S *s = static_cast<const S *>(src[q]) + (size_t)member * sbs[q];
    for (long long i = tid; i < n; i += kThreads) dst[off[q] + i] = s[i];
  }
  if (tid == 0)
    for (int q = 0; q <= L; ++q) rk[q] = r0[q];
  __syncthreads();
  if (!orth) return;
  for (int q = L - 1; q >= 1; --q) {
    const int r = rk[q], c = legs[q] * rk[q + 1];
    S *core = dst + off[q];
    // H = M^T (c x r, column-major): H[j + i c] = M[i, j] = core[i c + j] -- the same storage
    for (int idx = tid; idx < r * c; idx += kThreads) H[idx] = core[idx];
    __syncthreads();
    house_qr(H, c, r, tau, red);
    const int k = min(r, c);
    form_q(H, c, k, tau, Q);                      // Q: c x k
    // core q <- Q^T (k x c): core[kk c + j] = Q[j + kk c]
    for (int idx = tid; idx < k * c; idx += kThreads) core[idx] = Q[idx];
    // core q-1 (rows = r_{q-1} legs_{q-1}, cols r) <- core q-1 R^T (cols k); R = k x r upper
    // (in H: R[i, j] = H[i + j c] for i <= j)
    S *prev = dst + off[q - 1];
    const int pr = rk[q - 1] * legs[q - 1];
    // stage prev into Q's space is not needed: compute into the tail of Q (pr x k)
    S *tmp = Q + (size_t)c * k;
    for (int idx = tid; idx < pr * k; idx += kThreads) {
      const int row = idx / k, kk = idx % k;
      S acc = mk<S>(0.0, 0.0);
      for (int j = kk; j < r; ++j) acc = zfma(prev[(size_t)row * r + j], H[kk + (size_t)j * c], acc);   // R^T[j,kk] = R[kk,j]
      tmp[idx] = acc;
    }
    __syncthreads();
    for (int idx = tid; idx < pr * k; idx += kThreads) prev[idx] = tmp[idx];
    if (tid == 0) rk[q] = k;
    __syncthreads();
  }
}

// a2 for one site: T[(c,i),(w',r')] = sum G[c,w,r] x[r,j,r'] op[w,i,j,w'] with `rows` carry
// rows c (for window 2 the rows are (chi, pending digit), so the same formula applies)
template <typename S>
__device__ void contract(const Args &a, int rows, int d, int dj, int w, int w2, int r, int r2, const S *G, const S *X,
                         const S *O, S *T, S *X1, double *gsm) {
  const int n = w2 * r2;
  if constexpr (sizeof(S) == sizeof(double)) {    // real: X1 = G x as a CTA GEMM, then the operator core
    if (a.kind != TRUNCATE) {
      const int N = dj * r2;                      // X1[(c, w), (j, r')] = sum_r G[(c, w), r] x[r, (j, r')]
      cta_gemm<kThreads>(rows * w, N, r, [&](int i, int k) { return G[(size_t)i * r + k]; },
                         [&](int k, int j) { return X[(size_t)k * N + j]; },
                         [&](int i, int j, double v) { X1[(size_t)i * N + j] = v; }, gsm);
      __syncthreads();
      for (int idx = threadIdx.x; idx < rows * d * n; idx += kThreads) {
        const int rr2 = idx % r2, ww2 = (idx / r2) % w2, ii = (idx / n) % d, c = idx / (n * d);
        double acc = 0.0;
        for (int ww = 0; ww < w; ++ww) {
          if (a.kind == HADAMARD) {
            acc = fma(O[((size_t)ww * d + ii) * w2 + ww2], X1[(((size_t)c * w + ww) * dj + ii) * r2 + rr2], acc);
          } else {
            for (int jj = 0; jj < dj; ++jj)
              acc = fma(O[(((size_t)ww * d + ii) * dj + jj) * w2 + ww2], X1[(((size_t)c * w + ww) * dj + jj) * r2 + rr2], acc);
          }
        }
        T[idx] = acc;
      }
      __syncthreads();
      return;
    }
  }
  for (int idx = threadIdx.x; idx < rows * d * n; idx += kThreads) {
    const int rr2 = idx % r2, ww2 = (idx / r2) % w2, ii = (idx / n) % d, c = idx / (n * d);
    S acc = mk<S>(0.0, 0.0);
    if (a.kind == TRUNCATE) {
      for (int rr = 0; rr < r; ++rr) acc = zfma(G[(size_t)c * r + rr], X[((size_t)rr * dj + ii) * r2 + rr2], acc);
    } else if (a.kind == HADAMARD) {
      for (int ww = 0; ww < w; ++ww) {
        const S o = O[((size_t)ww * d + ii) * w2 + ww2];
        S t = mk<S>(0.0, 0.0);
        for (int rr = 0; rr < r; ++rr) t = zfma(G[((size_t)c * w + ww) * r + rr], X[((size_t)rr * d + ii) * r2 + rr2], t);
        acc = zfma(o, t, acc);
      }
    } else {
      for (int ww = 0; ww < w; ++ww)
        for (int jj = 0; jj < dj; ++jj) {
          const S o = O[(((size_t)ww * d + ii) * dj + jj) * w2 + ww2];
          S t = mk<S>(0.0, 0.0);
          for (int rr = 0; rr < r; ++rr)
            t = zfma(G[((size_t)c * w + ww) * r + rr], X[((size_t)rr * dj + jj) * r2 + rr2], t);
          acc = zfma(o, t, acc);
        }
    }
    T[idx] = acc;
  }
  __syncthreads();
}

// One CTA per member.  Window 1: site q's matrix is T (chi d_q) x (w' r').  Window 2
// (PAPER.md:266 N = 2): the carry keeps the pending digit, rows
// (chi_{q}, i_q), and absorbing site q+1 gives the super-core split as (chi d_q) x
// (d_{q+1} w' r') -- the same memory read with another row/column split; its rank is capped
// at w_{q+1} r_{q+1} (reading c-A35), and the last split leaves C_{L-1} = diag(s) V^H.
template <typename S>
__global__ void __launch_bounds__(kThreads, 1) k_zipup(Args a) {
  const int b = blockIdx.x, tid = threadIdx.x, L = a.L, L1 = L + 1;
  __shared__ double red[kWarps];
  __shared__ double s_sc[4];
  extern __shared__ __align__(16) unsigned char zsm_raw[];
  // real scalars (a.jreg): dynamic shared memory = [Rp (packed R; also the cta_gemm staging and
  // the Jacobi scratch, never live at the same time)] [Bk / Jacobi matrix, 128 x kLdA] [Ysm] [tau]
  double *Rp = reinterpret_cast<double *>(zsm_raw + a.jsm_off);
  double *Bk = Rp + kRpDoubles, *Ysm = Bk + kQBkDoubles, *tauq = Ysm + 16 * kYld;
  double *gsm = Rp;
  S *zsm = reinterpret_cast<S *>(zsm_raw);
  S *w0 = static_cast<S *>(a.ws) + (size_t)b * a.ws_member;
  S *Xo = w0, *Oo = Xo + a.xo_n, *G = Oo + a.oo_n, *T = G + a.g_n, *H = T + a.t_n, *Q = H + a.t_n,
    *tau = Q + 2 * a.t_n;
  if (a.smem) {                         // the member's matrices fit on chip (the Fourier chain does)
    T = zsm; H = T + a.t_n; Q = H + a.t_n; G = Q + 2 * a.t_n; tau = G + a.g_n;
  }
  char *iw = a.iws + (size_t)b * a.iws_member;
  double *sg = (double *)iw;                      // [pmax]
  double *tail = sg + a.pmax;                     // [pmax + 1]
  int *perm = (int *)(tail + a.pmax + 1);         // [pmax]
  int *xr = perm + a.pmax, *orr = xr + L1;        // [L+1] each
  const int ob = (a.op_batch == 1) ? 0 : b;
  const bool win2 = a.window == 2 && L >= 2;

  // ---- a1
  long long tph = clock64();
  if (a.xr_pre) {                                 // done by the fp64 path's k_orth (real scalars)
    for (int q = tid; q <= L; q += kThreads) {
      xr[q] = a.xr_pre[(size_t)b * L1 + q];
      orr[q] = (a.kind == TRUNCATE) ? 1 : a.orr_pre[(size_t)b * L1 + q];
    }
    if (a.op_batch == 1 && a.B > 1) Oo = static_cast<S *>(a.ws) + a.xo_n;   // shared operator: member 0's slot
    __syncthreads();
  } else {
    int legs[64];
    for (int q = 0; q < L; ++q) legs[q] = a.dj[q];
    orth_operand<S>(a, a.xsrc, a.x_bs, b, legs, a.xr0, a.xoff, Xo, xr, true, H, Q, tau, red);
    if (a.kind != TRUNCATE) {
      for (int q = 0; q < L; ++q) legs[q] = (a.kind == MATVEC) ? a.d[q] * a.dj[q] : a.d[q];
      orth_operand<S>(a, a.osrc, a.o_bs, ob, legs, a.or0, a.ooff, Oo, orr, a.orth_op != 0, H, Q, tau, red);
    } else if (tid == 0) {
      for (int q = 0; q <= L; ++q) orr[q] = 1;
    }
    __syncthreads();
  }
  if (tid == 0) G[0] = mk<S>(1.0, 0.0);
  if (tid == 0 && a.cycles) a.cycles[(size_t)b * L * 4 + 3] = clock64() - tph;
  __syncthreads();
  int rows = 1;                                   // carry rows: chi (window 1) or chi d_pending (window 2)
  int chi = 1;                                    // bond of the next output core
  int s0 = 0;
  if (win2) {                                     // the first site contracted exactly into the carry
    contract<S>(a, 1, a.d[0], a.dj[0], orr[0], orr[1], xr[0], xr[1], G, Xo + a.xoff[0], Oo + a.ooff[0], T, H, gsm);
    const int n0 = a.d[0] * orr[1] * xr[1];
    for (int i = tid; i < n0; i += kThreads) G[i] = T[i];
    rows = a.d[0];
    s0 = 1;
    __syncthreads();
  }
  tph = clock64();
  for (int st = s0; st < L; ++st) {
    // absorb site st; the split emits output core q (q = st for window 1, st - 1 for window 2)
    const int q = win2 ? st - 1 : st;
    const int d = a.d[st], dj = a.dj[st];
    const int w = orr[st], w2 = orr[st + 1], r = xr[st], r2 = xr[st + 1];
    contract<S>(a, rows, d, dj, w, w2, r, r2, G, Xo + a.xoff[st], Oo + a.ooff[st], T, H, gsm);
    const int m = win2 ? rows : rows * d;         // split: rows (chi, i_q) ...
    const int n = win2 ? d * w2 * r2 : w2 * r2;   // ... columns (window 2: i_{q+1}, w', r')
    S *Cq = static_cast<S *>(a.Cq[q]) + (size_t)b * a.Cq_bs[q];
    if (tid == 0 && a.cycles) a.cycles[((size_t)b * L + q) * 4 + 0] = clock64() - tph;
    tph = clock64();
    // ---- a7: last site (window 1)
    if (!win2 && q == L - 1) {
      double sq = 0.0;
      for (int i = tid; i < m * n; i += kThreads) { Cq[i] = T[i]; sq += abs2(T[i]); }
      sq = block_sum(sq, red);
      if (tid == 0) {
        a.norm2[b] = sq;
        a.delta2[(size_t)b * L + q] = 0.0;
        a.yr[(size_t)b * L1 + L] = 1;
        if (L == 1) a.yr[(size_t)b * L1] = 1;
        if (a.sweeps) a.sweeps[(size_t)b * L + q] = 0;
        if (!isfinite(sq)) atomicOr(a.status, 1);
      }
      return;
    }
    // ---- a3: A (m x p, column-major, ld m)
    int p;
    S *A = Q;                                     // reuse: Q is free between a1 and here
    bool in_js = false;                           // real: A = R^T already in the Jacobi matrix Bk
    if constexpr (sizeof(S) == sizeof(double)) {
      if (a.jreg && m <= n && m <= kSmall) {      // the fp64 path's blocked QR (qr_small.cuh)
        p = m;
        qr_of_TH(reinterpret_cast<const double *>(T), m, n, Rp, Bk, tauq, Ysm);
        __syncthreads();
        const int mp = (m <= 32) ? 32 : (m <= 64) ? 64 : 128;
        const int pp = 2 * kWarps * ((p <= 2 * kWarps) ? 1 : (p <= 4 * kWarps) ? 2 : (p <= 8 * kWarps) ? 4 : 8);
        for (int idx = tid; idx < pp * mp; idx += kThreads) {   // A = R^T, zero-padded, ld kLdA
          const int j = idx / mp, row = idx % mp;
          Bk[(size_t)j * kLdA + row] = (row < m && j < p && row >= j) ? Rp[rp_idx(j, row, m)] : 0.0;
        }
        in_js = true;
      }
    }
    if (in_js) {
    } else if (m <= n) {
      p = m;
      for (int idx = tid; idx < m * n; idx += kThreads) H[idx] = conj(T[idx]);   // T^H column-major (n x m)
      __syncthreads();
      house_qr<S>(H, n, m, tau, red);
      for (int idx = tid; idx < m * m; idx += kThreads) {       // A = R^H: A[i, j] = conj(R[j, i]), i >= j
        const int j = idx / m, i = idx % m;
        A[idx] = (i >= j) ? conj(H[j + (size_t)i * n]) : mk<S>(0.0, 0.0);
      }
    } else {
      p = n;
      for (int idx = tid; idx < m * n; idx += kThreads) {
        const int j = idx / m, i = idx % m;
        A[idx] = T[(size_t)i * n + j];
      }
    }
    __syncthreads();
    if (tid == 0 && a.cycles) a.cycles[((size_t)b * L + q) * 4 + 1] = clock64() - tph;
    tph = clock64();
    // ---- a4
    int sweeps = -1;
    if constexpr (sizeof(S) == sizeof(double)) {
      if (a.jreg && m <= 128 && p <= 128) {      // the fp64 path's register-blocked Jacobi
        double *Js = Bk;
        double *jscr = Rp;                       // Rp is free once A = R^T sits in Bk
        int *jflag = reinterpret_cast<int *>(jscr + 1024);
        if (!in_js) {
          const int mp = (m <= 32) ? 32 : (m <= 64) ? 64 : 128;
          const int pp = 2 * kWarps * ((p <= 2 * kWarps) ? 1 : (p <= 4 * kWarps) ? 2 : (p <= 8 * kWarps) ? 4 : 8);
          for (int idx = tid; idx < pp * mp; idx += kThreads) {   // zero-padded, ld kLdA
            const int j = idx / mp, row = idx % mp;
            Js[(size_t)j * kLdA + row] = (row < m && j < p) ? (double)A[(size_t)j * m + row] : 0.0;
          }
        }
        __syncthreads();
        sweeps = jacobi_dispatch<kWarps>(Js, m, p, jflag, jscr, noise_ok(a.eps, p));
        for (int idx = tid; idx < p * m; idx += kThreads) {
          const int j = idx / m, row = idx % m;
          A[idx] = Js[(size_t)j * kLdA + row];
        }
        __syncthreads();
      }
    }
    if (sweeps < 0) sweeps = jacobi<S>(A, m, p, noise_ok(a.eps, p) ? DBL_EPSILON * DBL_EPSILON : 0.0, red);
    for (int j = tid >> 5; j < p; j += kWarps) {
      double sq = 0.0;
      for (int i = tid & 31; i < m; i += 32) sq += abs2(A[(size_t)j * m + i]);
      sq = warp_sum(sq);
      if ((tid & 31) == 0) {
        if (!isfinite(sq)) { atomicOr(a.status, 1); sq = 0.0; }
        sg[j] = sq;
      }
    }
    __syncthreads();
    for (int j = tid; j < p; j += kThreads) {
      const double sj = sg[j];
      int rank = 0;
      for (int l = 0; l < p; ++l) rank += (sg[l] > sj) || (sg[l] == sj && l < j);
      perm[rank] = j;
    }
    __syncthreads();
    if (tid == 0 && a.cycles) a.cycles[((size_t)b * L + q) * 4 + 2] = clock64() - tph;
    tph = clock64();
    // ---- a5
    if (tid == 0) {
      double acc = 0.0;
      tail[p] = 0.0;
      for (int jj = p - 1; jj >= 0; --jj) { acc += sg[perm[jj]]; tail[jj] = acc; }
      const double tot = acc, thr = a.eps * a.eps * tot;
      int k = p;
      for (int kk = 1; kk <= p; ++kk)
        if (tail[kk] <= thr) { k = kk; break; }
      if (a.max_rank > 0) k = min(k, a.max_rank);
      if (win2) k = min(k, xr[q + 1] * orr[q + 1]);            // c-A35: exact rank at bond q+1
      if (tot == 0.0) k = 1;
      k = max(k, 1);
      s_sc[0] = (double)k;
      s_sc[1] = tail[k];
      if (sweeps >= kMaxSweeps) atomicOr(a.status, 2);
    }
    __syncthreads();
    const int k = (int)s_sc[0];
    // ---- a6: U columns, emit, carry
    for (int idx = tid; idx < k * m; idx += kThreads) {
      const int kk = idx / m, i = idx % m;
      const int j = perm[kk];
      const double s2 = sg[j];
      S *col = A + (size_t)j * m;
      col[i] = (s2 > 0.0) ? scl(1.0 / sqrt(s2), col[i]) : mk<S>((i == kk) ? 1.0 : 0.0, 0.0);
    }
    __syncthreads();
    for (int idx = tid; idx < m * k; idx += kThreads) {
      const int i = idx / k, kk = idx % k;
      Cq[idx] = A[(size_t)perm[kk] * m + i];
    }
    if (a.sigma) {
      double *so = a.sigma + ((size_t)b * (L - 1) + q) * a.sigma_stride;
      for (int jj = tid; jj < a.sigma_stride; jj += kThreads) so[jj] = (jj < p) ? sqrt(sg[perm[jj]]) : 0.0;
    }
    if (tid == 0) {
      if (a.sweeps) a.sweeps[(size_t)b * L + q] = sweeps;
      a.yr[(size_t)b * L1 + q + 1] = k;
      if (q == 0) a.yr[(size_t)b * L1] = 1;
      a.delta2[(size_t)b * L + q] = s_sc[1];
    }
    // G[kk, col] = sum_i conj(U[i, kk]) T[i, col]   (k x n)
    if constexpr (sizeof(S) == sizeof(double)) {
      cta_gemm<kThreads>(k, n, m, [&](int kk, int i) { return (double)A[(size_t)perm[kk] * m + i]; },
                         [&](int i, int col) { return (double)T[(size_t)i * n + col]; },
                         [&](int kk, int col, double v) { G[(size_t)kk * n + col] = v; }, gsm);
    } else {
      for (int idx = tid; idx < k * n; idx += kThreads) {
        const int kk = idx / n, col = idx % n;
        const S *u = A + (size_t)perm[kk] * m;
        S acc = mk<S>(0.0, 0.0);
        for (int i = 0; i < m; ++i) acc = cfma(u[i], T[(size_t)i * n + col], acc);
        G[idx] = acc;
      }
    }
    __syncthreads();
    if (win2 && st == L - 1) {                    // fully decomposed: C_{L-1} = diag(s) V^H (k, d, 1)
      S *Cl = static_cast<S *>(a.Cq[L - 1]) + (size_t)b * a.Cq_bs[L - 1];
      double sq = 0.0;
      for (int i = tid; i < k * n; i += kThreads) { Cl[i] = G[i]; sq += abs2(G[i]); }
      sq = block_sum(sq, red);
      if (tid == 0) {
        a.norm2[b] = sq;
        a.delta2[(size_t)b * L + L - 1] = 0.0;
        a.yr[(size_t)b * L1 + L] = 1;
        if (a.sweeps) a.sweeps[(size_t)b * L + L - 1] = 0;
        if (!isfinite(sq)) atomicOr(a.status, 1);
      }
      return;
    }
    chi = k;
    rows = win2 ? k * d : k;
    if (tid == 0 && a.cycles && q > 0) a.cycles[((size_t)b * L + q) * 4 + 3] = clock64() - tph;
    tph = clock64();
  }
  (void)chi;
}

}  // namespace cplx

static void member_sizes(const Shape &S, int window, long long &zmember, long long &imember, long long &xo,
                         long long &oo, long long &gn, long long &tn, int &pmax) {
  xo = S.xoff[S.L];
  oo = std::max<long long>(1, S.ooff[S.L]);
  gn = S.g_elems;
  tn = S.t_elems;
  pmax = 1;
  long long core_max = 1;
  for (int q = 0; q < S.L; ++q) {
    const long long m = (long long)S.cap[q] * S.d[q], n = (long long)S.orr[q + 1] * S.xr[q + 1];
    pmax = (int)std::max<long long>(pmax, std::max(m, n));
    core_max = std::max(core_max, (long long)S.xr[q] * S.dj[q] * S.xr[q + 1]);
    const long long oc = (S.kind == MATVEC) ? (long long)S.orr[q] * S.d[q] * S.dj[q] * S.orr[q + 1]
                                            : (long long)S.orr[q] * S.d[q] * S.orr[q + 1];
    core_max = std::max(core_max, oc);
  }
  for (int q = 0; q < S.L; ++q) {        // X1 = G x staged in the H region during the contraction
    const long long rows = (window == 2 && q > 0) ? (long long)S.cap[q - 1] * S.d[q - 1] : (long long)S.cap[q];
    const long long w = (S.kind == TRUNCATE) ? 1 : S.orr[q];
    tn = std::max(tn, std::max(rows, 1LL) * w * S.dj[q] * S.xr[q + 1]);
  }
  if (window == 2) {                    // super-core (chi d_q) x (d_{q+1} w' r') and its carry
    for (int st = 1; st < S.L; ++st) {
      const long long m = (long long)S.cap[st - 1] * S.d[st - 1];
      const long long n = (long long)S.d[st] * S.orr[st + 1] * S.xr[st + 1];
      tn = std::max(tn, m * n);
      gn = std::max(gn, (long long)S.cap[st] * n);
      pmax = (int)std::max<long long>(pmax, std::max(m, n));
    }
    gn = std::max(gn, (long long)S.d[0] * S.orr[1] * S.xr[1]);
    tn = std::max(tn, (long long)S.d[0] * S.orr[1] * S.xr[1]);
  }
  tn = std::max(tn, core_max);
  // regions: Xo, Oo, G, T (tn), H (tn), Q (2 tn: Q / A and the a1 product), tau (pmax)
  zmember = xo + oo + gn + tn + tn + 2 * tn + std::max<long long>(pmax, 64);
  zmember = (zmember + 15) & ~15LL;
  imember = 8LL * (3LL * pmax + 1) + 4LL * (2LL * (S.L + 1)) + 256;
  imember = (imember + 255) & ~255LL;
}

size_t member_workspace_bytes(const Shape &S, int elem_bytes, int window) {
  long long zm, im, xo, oo, gn, tn;
  int pmax;
  member_sizes(S, window, zm, im, xo, oo, gn, tn, pmax);
  // + the a1 ranks of the real path's k_orth pre-pass ([B][L+1] for x and for the operator)
  return (size_t)S.B * (size_t)zm * elem_bytes + (size_t)S.B * (size_t)im + 256 +
         (elem_bytes == 8 ? 2 * (size_t)S.B * (S.L + 1) * sizeof(int) + 256 : 0);
}

qtt_status_t member_zipup(const Shape &S, const qtt_trains_t *op, const qtt_trains_t *x, uint32_t flags,
                          const LargeIO &io, void *workspace, size_t workspace_bytes, cudaStream_t s,
                          long long *cycles, bool complex_dt, int window, void *const *events) {
  if (S.L > 64) { set_error("per-member path: n_sites > 64"); return QTT_EUNSUPPORTED; }
  const int elem = complex_dt ? 16 : 8;
  const size_t need = member_workspace_bytes(S, elem, window);
  if (!workspace || workspace_bytes < need) {
    set_error("workspace %zu bytes < required %zu", workspace_bytes, need);
    return QTT_ECAPACITY;
  }
  cplx::Args a;
  memset(&a, 0, sizeof(a));
  a.L = S.L; a.B = S.B; a.kind = S.kind; a.op_batch = op ? op->batch : 1;
  for (int q = 0; q < S.L; ++q) {
    a.d[q] = S.d[q]; a.dj[q] = S.dj[q];
    a.xsrc[q] = x->cores[q];
    a.x_bs[q] = (long long)x->ranks[q] * x->d_out[q] * x->ranks[q + 1];
    if (op) {
      a.osrc[q] = op->cores[q];
      a.o_bs[q] = (long long)op->ranks[q] * op->d_out[q] * (op->n_legs == 2 ? op->d_in[q] : 1) * op->ranks[q + 1];
    }
    a.Cq[q] = io.out->cores[q];
    a.Cq_bs[q] = (long long)io.out->ranks[q] * S.d[q] * io.out->ranks[q + 1];
  }
  for (int q = 0; q <= S.L; ++q) {
    a.xr0[q] = S.xr[q]; a.or0[q] = S.orr[q]; a.cap[q] = S.cap[q];
    a.xoff[q] = S.xoff[q]; a.ooff[q] = S.ooff[q];
  }
  long long zm, im, xo, oo, gn, tn;
  int pmax;
  member_sizes(S, window, zm, im, xo, oo, gn, tn, pmax);
  a.ws = workspace;
  a.ws_member = zm;
  a.xo_n = xo; a.oo_n = oo; a.g_n = gn; a.t_n = tn;
  a.iws = (char *)workspace + (size_t)S.B * zm * elem;
  a.iws_member = im;
  a.pmax = pmax;
  a.yr = io.out_ranks; a.delta2 = io.delta2; a.norm2 = io.norm2; a.sigma = io.sigma;
  a.sigma_stride = io.sigma_stride; a.sweeps = io.sweeps; a.status = io.status;
  a.eps = io.eps; a.max_rank = io.max_rank;
  a.orth_op = (flags & QTT_NO_OPERATOR_ORTH) ? 0 : 1;
  a.cycles = cycles;
  a.window = window;
  // a1 by the fp64 path's register-resident k_orth when every core fits its shared-memory
  // staging budget; otherwise (bonds wider than k_orth stages) the kernel's own global-memory
  // orth_operand runs (xr_pre stays NULL)
  if (!complex_dt && a1_fits(S, false)) {
    int *ranks_pre = (int *)((char *)workspace + (size_t)S.B * zm * elem + (size_t)S.B * im + 256);
    a.xr_pre = ranks_pre;
    a.orr_pre = ranks_pre + (size_t)S.B * (S.L + 1);
    qtt_status_t st = orth_prepass(S, op, x, flags, (double *)workspace, (double *)workspace + xo, zm,
                                   (int *)a.xr_pre, (int *)a.orr_pre, s);
    if (st != QTT_OK) return st;
  }
  // diag events: [0] before a1 (caller), [1] after the a1 pre-pass, [2] before k_zipup, [3] after (caller)
  if (events) QTT_CUDA_TRY(cudaEventRecord((cudaEvent_t)events[1], s));
  QTT_CUDA_TRY(cudaMemsetAsync(io.status, 0, sizeof(int32_t), s));
  if (events) QTT_CUDA_TRY(cudaEventRecord((cudaEvent_t)events[2], s));
  size_t smem = (size_t)(4 * tn + gn + std::max(pmax, 64)) * elem;
  if (complex_dt) {                     // the member's matrices on chip when they fit
    a.jreg = 0;
    a.smem = smem <= 200 * 1024 ? 1 : 0;
    a.jsm_off = 0;
    if (!a.smem) smem = 0;
  } else {                              // real: blocked QR + register Jacobi working set on chip
    a.jreg = 1;
    a.smem = 0;
    a.jsm_off = 0;
    smem = (size_t)(kRpDoubles + kQBkDoubles + 16 * kYld + kSmall) * sizeof(double);
  }
  if (complex_dt) {       // dynamic-smem opt-in every call (per-device attribute; thread-safe)
    if (a.smem)
      QTT_CUDA_TRY(cudaFuncSetAttribute(cplx::k_zipup<cplx::Z>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cplx::k_zipup<cplx::Z><<<S.B, kThreads, smem, s>>>(a);
  } else {
    QTT_CUDA_TRY(cudaFuncSetAttribute(cplx::k_zipup<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cplx::k_zipup<double><<<S.B, kThreads, smem, s>>>(a);
  }
  QTT_CUDA_TRY(cudaGetLastError());
  return QTT_OK;
}

}  // namespace qtt

// ======================================================================= f3: variational
// Single-site variational refinement seeded by a zip-up result (Eq.
// variational 294; reading c-A36).  One CTA per member:
//   C right-orthonormalised (centre at 0); right environments Re[q] (c, w, r);
//   sweep: q = 0..L-1: C_q = sum Le[q] W_q x_q Re[q+1]; QR moves the centre right and Le[q+1]
//   is built from the new left-orthonormal C_q; then q = L-1..0 with LQ / Re[q].
//   |C_q|^2 after every update goes to center_norm2 (|O - C|^2 = |O|^2 - |C_q|^2).
namespace qtt {
namespace cplx {

struct VarArgs {
  int L, B, kind, op_batch, sweeps;
  int ncores, max_rank;               // 1: single-site; 2: two-site super-cores (reading c-A37)
  double eps;                         // two-site split truncation (SPEC.md:299 rule, eps = cutoff)
  int d[64], dj[64], xr[65], orr[65], cap[65];
  const double *x[64];
  const double *op[64];
  long long x_bs[64], o_bs[64];
  const double *sd[64];               // seed slots (may alias c)
  long long sd_bs[64];
  const int *sd_ranks;                // device [B][L+1] the seed's ranks
  double *c[64];
  long long c_bs[64];
  int *c_ranks;                       // device [B][L+1] out: ranks after the sweeps
  double *norms;                      // device [B][sweeps * 2L]
  int *status;
  double *ws;
  long long ws_member;
  long long coff[65], eoff[65];       // per-member offsets: C slots (capacity), environments
  long long e_n, s_n;                 // environment region (each of Le, Re) and scratch sizes
  int pmax;                           // >= every split's min(m, n) and row count
};

// W[w, i, j, w'] of the operator (Hadamard: A[w, i, w'] on i == j; truncate: identity)
__device__ __forceinline__ double opval(const VarArgs &a, const double *O, int q, int w, int i, int j, int w2,
                                        int wr2) {
  if (a.kind == MATVEC) return O[(((size_t)w * a.d[q] + i) * a.dj[q] + j) * wr2 + w2];
  if (a.kind == HADAMARD) return (i == j) ? O[((size_t)w * a.d[q] + i) * wr2 + w2] : 0.0;
  return (i == j) ? 1.0 : 0.0;
}

// X2[c, i, w', r'] = sum_{w, r, j} Le[c, w, r] W[w, i, j, w'] x[r, j, r']   (c < rc)
__device__ void env_apply_left(const VarArgs &a, int q, int rc, const double *Le, const double *X,
                               const double *O, double *X1, double *X2, double *gsm) {
  const int tid = threadIdx.x;
  const int d = a.d[q], dj = a.dj[q];
  const int w = (a.kind == TRUNCATE) ? 1 : a.orr[q], w2 = (a.kind == TRUNCATE) ? 1 : a.orr[q + 1];
  const int r = a.xr[q], r2 = a.xr[q + 1];
  // X1[(c, w), (j, r')] = sum_r Le[(c, w), r] x[r, (j, r')]   (CTA GEMM, smem-staged tiles)
  {
    const int N = dj * r2;
    cta_gemm<kThreads>(rc * w, N, r, [&](int i, int k) { return Le[(size_t)i * r + k]; },
                       [&](int k, int j) { return X[(size_t)k * N + j]; },
                       [&](int i, int j, double v) { X1[(size_t)i * N + j] = v; }, gsm);
  }
  __syncthreads();
  // X2[c, i, w', r'] = sum_{w, j} X1[c, w, j, r'] W[w, i, j, w']
  for (int idx = tid; idx < rc * d * w2 * r2; idx += kThreads) {
    const int rr2 = idx % r2, ww2 = (idx / r2) % w2, ii = (idx / (r2 * w2)) % d, c = idx / (r2 * w2 * d);
    double s = 0.0;
    for (int ww = 0; ww < w; ++ww)
      for (int jj = 0; jj < dj; ++jj) {
        if (a.kind != MATVEC && jj != ii) continue;
        s = fma(X1[(((size_t)c * w + ww) * dj + jj) * r2 + rr2], opval(a, O, q, ww, ii, jj, ww2, w2), s);
      }
    X2[idx] = s;
  }
  __syncthreads();
}

// Re_new[c, w, r] = sum C[c, i, c'] W[w, i, j, w'] x[r, j, r'] Re[c', w', r']
__device__ void env_right(const VarArgs &a, int q, int rc, int rc2, const double *C, const double *Re,
                          const double *X, const double *O, double *Y1, double *Y2, double *Rn, double *gsm) {
  const int tid = threadIdx.x;
  const int d = a.d[q], dj = a.dj[q];
  const int w = (a.kind == TRUNCATE) ? 1 : a.orr[q], w2 = (a.kind == TRUNCATE) ? 1 : a.orr[q + 1];
  const int r = a.xr[q], r2 = a.xr[q + 1];
  // Y1[(c, i), (w', r')] = sum_{c'} C[(c, i), c'] Re[c', (w', r')]
  {
    const int N = w2 * r2;
    cta_gemm<kThreads>(rc * d, N, rc2, [&](int i, int k) { return C[(size_t)i * rc2 + k]; },
                       [&](int k, int j) { return Re[(size_t)k * N + j]; },
                       [&](int i, int j, double v) { Y1[(size_t)i * N + j] = v; }, gsm);
  }
  __syncthreads();
  // Y2[c, w, j, r'] = sum_{i, w'} Y1[c, i, w', r'] W[w, i, j, w']
  for (int idx = tid; idx < rc * w * dj * r2; idx += kThreads) {
    const int rr2 = idx % r2, jj = (idx / r2) % dj, ww = (idx / (r2 * dj)) % w, c = idx / (r2 * dj * w);
    double s = 0.0;
    for (int ii = 0; ii < d; ++ii) {
      if (a.kind != MATVEC && ii != jj) continue;
      for (int ww2 = 0; ww2 < w2; ++ww2)
        s = fma(Y1[(((size_t)c * d + ii) * w2 + ww2) * r2 + rr2], opval(a, O, q, ww, ii, jj, ww2, w2), s);
    }
    Y2[idx] = s;
  }
  __syncthreads();
  // Rn[(c, w), r] = sum_{(j, r')} Y2[(c, w), (j, r')] x[r, (j, r')]
  {
    const int K = dj * r2;
    cta_gemm<kThreads>(rc * w, r, K, [&](int i, int k) { return Y2[(size_t)i * K + k]; },
                       [&](int k, int j) { return X[(size_t)j * K + k]; },
                       [&](int i, int j, double v) { Rn[(size_t)i * r + j] = v; }, gsm);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 1) k_variational(VarArgs a) {
  const int b = blockIdx.x, tid = threadIdx.x, L = a.L;
  __shared__ double red[kWarps];
  __shared__ double gsm[2 * 16 * 64];            // cta_gemm staging
  __shared__ int cr[65];
  __shared__ double s_k[2];
  double *w0 = a.ws + (size_t)b * a.ws_member;
  double *Cw = w0, *Le = Cw + a.coff[L], *Re = Le + a.e_n, *S1 = Re + a.e_n, *S2 = S1 + a.s_n, *S3 = S2 + a.s_n,
         *S4 = S3 + a.s_n, *S5 = S4 + a.s_n, *tau = S5 + a.s_n, *sg = tau + a.pmax;
  int *perm = reinterpret_cast<int *>(sg + a.pmax);
  const int ob = (a.op_batch == 1) ? 0 : b;
  for (int q = tid; q <= L; q += kThreads) cr[q] = a.sd_ranks[(size_t)b * (L + 1) + q];
  __syncthreads();
  // the seed into the workspace, packed at its ranks (read completely before c is written:
  // the seed may alias the output slots)
  for (int q = 0; q < L; ++q) {
    const long long n = (long long)cr[q] * a.d[q] * cr[q + 1];
    const double *src = a.sd[q] + (size_t)b * a.sd_bs[q];
    for (long long i = tid; i < n; i += kThreads) Cw[a.coff[q] + i] = src[i];
  }
  __syncthreads();
  auto Xq = [&](int q) { return a.x[q] + (size_t)b * a.x_bs[q]; };
  auto Oq = [&](int q) { return a.op[q] ? a.op[q] + (size_t)ob * a.o_bs[q] : (const double *)nullptr; };
  // centre from q to q-1: C_q^T = Q R (thin, k = min(r, c) -- the bond shrinks when the core
  // cannot be row-orthonormal, as numpy's reduced QR in the oracle), C_q <- Q^T, C_{q-1} <- C_{q-1} R^T
  auto move_left = [&](int q) {
    const int r = cr[q], c = a.d[q] * cr[q + 1], k = min(r, c);
    double *core = Cw + a.coff[q];
    for (int idx = tid; idx < r * c; idx += kThreads) S1[idx] = core[idx];   // C_q^T, column-major (c x r)
    __syncthreads();
    house_qr<double>(S1, c, r, tau, red);
    form_q<double>(S1, c, k, tau, S2);
    for (int idx = tid; idx < k * c; idx += kThreads) core[idx] = S2[idx];
    double *prev = Cw + a.coff[q - 1];
    const int pr = cr[q - 1] * a.d[q - 1];
    for (int idx = tid; idx < pr * k; idx += kThreads) {
      const int row = idx / k, kk = idx % k;
      double sacc = 0.0;
      for (int j2 = kk; j2 < r; ++j2) sacc = fma(prev[(size_t)row * r + j2], S1[kk + (size_t)j2 * c], sacc);
      S3[idx] = sacc;
    }
    __syncthreads();
    for (int idx = tid; idx < pr * k; idx += kThreads) prev[idx] = S3[idx];
    if (tid == 0) cr[q] = k;
    __syncthreads();
  };
  // centre from q to q+1: C_q = Q R (rows = cr[q] d_q), C_{q+1} <- R C_{q+1}
  auto move_right = [&](int q) {
    const int rows = cr[q] * a.d[q], kc = cr[q + 1], k = min(rows, kc);
    double *C = Cw + a.coff[q];
    for (int idx = tid; idx < rows * kc; idx += kThreads) S1[(idx % kc) * rows + idx / kc] = C[idx];
    __syncthreads();
    house_qr<double>(S1, rows, kc, tau, red);
    form_q<double>(S1, rows, k, tau, S2);
    for (int idx = tid; idx < rows * k; idx += kThreads) C[idx] = S2[(idx % k) * rows + idx / k];
    double *Cn = Cw + a.coff[q + 1];
    const int cols = a.d[q + 1] * cr[q + 2];
    for (int idx = tid; idx < k * cols; idx += kThreads) {
      const int i2 = idx / cols, j2 = idx % cols;
      double sacc = 0.0;
      for (int l = i2; l < kc; ++l) sacc = fma(S1[i2 + (size_t)l * rows], Cn[(size_t)l * cols + j2], sacc);
      S3[idx] = sacc;
    }
    __syncthreads();
    for (int idx = tid; idx < k * cols; idx += kThreads) Cn[idx] = S3[idx];
    if (tid == 0) cr[q + 1] = k;
    __syncthreads();
  };
  for (int q = L - 1; q >= 1; --q) move_left(q);  // right-orthonormalise the seed: centre at site 0
  // environments
  if (tid == 0) { Le[a.eoff[0]] = 1.0; Re[a.eoff[L]] = 1.0; }
  __syncthreads();
  for (int q = L - 1; q >= 1; --q)
    env_right(a, q, cr[q], cr[q + 1], Cw + a.coff[q], Re + a.eoff[q + 1], Xq(q), Oq(q), S1, S2, Re + a.eoff[q], gsm);
  int cnt = 0;
  auto update = [&](int q) {                      // C_q = sum Le[q] W_q x_q Re[q+1]   (Eq. variational)
    env_apply_left(a, q, cr[q], Le + a.eoff[q], Xq(q), Oq(q), S1, S2, gsm);
    const int w2 = (a.kind == TRUNCATE) ? 1 : a.orr[q + 1], r2 = a.xr[q + 1], rc2 = cr[q + 1], d = a.d[q];
    double *C = Cw + a.coff[q];
    {  // C[(c, i), c'] = sum_{(w', r')} X2[(c, i), (w', r')] Re[c', (w', r')]
      const int K = w2 * r2;
      const double *R1 = Re + a.eoff[q + 1];
      cta_gemm<kThreads>(cr[q] * d, rc2, K, [&](int i, int k) { return S2[(size_t)i * K + k]; },
                         [&](int k, int j) { return R1[(size_t)j * K + k]; },
                         [&](int i, int j, double v) { C[(size_t)i * rc2 + j] = v; }, gsm);
    }
    __syncthreads();
    double sq = 0.0;
    for (int idx = tid; idx < cr[q] * d * rc2; idx += kThreads) sq = fma(C[idx], C[idx], sq);
    sq = block_sum(sq, red);
    if (tid == 0) {
      a.norms[(size_t)b * a.sweeps * 2 * L + cnt] = sq;
      if (!isfinite(sq)) atomicOr(a.status, 1);
    }
    ++cnt;
    __syncthreads();
  };
  // ---- two-site super-cores (ncores = 2, reading c-A37)
  // split(q): S[(c, i), (i', a)] = Le[q] W_q x_q W_{q+1} x_{q+1} Re[q+2] (into S1, row-major
  // m x n), SVD by Householder QR + one-sided Jacobi (as the zip-up's a3/a4), truncation by the
  // SPEC.md:299 rule (eps, max_rank, output capacity); C_q <- U_k, C_{q+1} <- U_k^T S =
  // diag(s_k) V_k^T (the centre sits at q+1).  Records |S_k|^2 = sum_{j<=k} s_j^2.
  auto split = [&](int q) {
    // X2[(c, i), (w', r')] from Le[q]  (S2; S1 scratch)
    env_apply_left(a, q, cr[q], Le + a.eoff[q], Xq(q), Oq(q), S1, S2, gsm);
    // Z[(c, i), i', (w'', r'')] = site q+1 absorbed with X2 as its left environment  (S3; S4 scratch)
    const int rc = cr[q] * a.d[q];
    env_apply_left(a, q + 1, rc, S2, Xq(q + 1), Oq(q + 1), S4, S3, gsm);
    const int w3 = (a.kind == TRUNCATE) ? 1 : a.orr[q + 2], r3 = a.xr[q + 2], a3 = cr[q + 2], d1 = a.d[q + 1];
    {  // M[(c, i, i'), a''] = sum_{(w'', r'')} Z[(c, i, i'), (w'', r'')] Re[q+2][a'', (w'', r'')]   (S1)
      const int K = w3 * r3;
      const double *R2 = Re + a.eoff[q + 2];
      cta_gemm<kThreads>(rc * d1, a3, K, [&](int i, int k) { return S3[(size_t)i * K + k]; },
                         [&](int k, int j) { return R2[(size_t)j * K + k]; },
                         [&](int i, int j, double v) { S1[(size_t)i * a3 + j] = v; }, gsm);
    }
    __syncthreads();
    const int m = rc, n = d1 * a3;
    int p;
    double *A = S4;                              // m x p, column-major
    if (m <= n) {                                // R of M^T: M = R^T Q^T, A = R^T (lower triangular)
      p = m;
      for (int idx = tid; idx < m * n; idx += kThreads) S5[idx] = S1[idx];   // M^T column-major (n x m)
      __syncthreads();
      house_qr<double>(S5, n, m, tau, red);
      for (int idx = tid; idx < m * m; idx += kThreads) {
        const int j = idx / m, i = idx % m;
        A[idx] = (i >= j) ? S5[j + (size_t)i * n] : 0.0;
      }
    } else {
      p = n;
      for (int idx = tid; idx < m * n; idx += kThreads) {
        const int j = idx / m, i = idx % m;
        A[idx] = S1[(size_t)i * n + j];
      }
    }
    __syncthreads();
    const int sweeps_done = jacobi<double>(A, m, p, noise_ok(a.eps, p) ? DBL_EPSILON * DBL_EPSILON : 0.0, red);
    for (int j = tid >> 5; j < p; j += kWarps) {
      double sq = 0.0;
      for (int i = tid & 31; i < m; i += 32) sq = fma(A[(size_t)j * m + i], A[(size_t)j * m + i], sq);
      sq = warp_sum(sq);
      if ((tid & 31) == 0) sg[j] = isfinite(sq) ? sq : 0.0;
      if ((tid & 31) == 0 && !isfinite(sq)) atomicOr(a.status, 1);
    }
    __syncthreads();
    for (int j = tid; j < p; j += kThreads) {
      const double sj = sg[j];
      int rank = 0;
      for (int l = 0; l < p; ++l) rank += (sg[l] > sj) || (sg[l] == sj && l < j);
      perm[rank] = j;
    }
    __syncthreads();
    if (tid == 0) {                              // SPEC.md:299, tails summed smallest first
      double acc = 0.0;
      for (int jj = p - 1; jj >= 0; --jj) acc += sg[perm[jj]];
      const double tot = acc, thr = a.eps * a.eps * tot;
      int k = p;
      double tl = 0.0;
      for (int kk = p - 1; kk >= 1; --kk) {      // tail[kk] = sum_{j >= kk} (sorted)
        tl += sg[perm[kk]];
        if (tl <= thr) k = kk;
      }
      if (a.max_rank > 0) k = min(k, a.max_rank);
      k = min(k, a.cap[q + 1]);
      if (tot == 0.0) k = 1;
      k = max(k, 1);
      double kept = 0.0;
      for (int jj = 0; jj < k; ++jj) kept += sg[perm[jj]];
      s_k[0] = (double)k;
      s_k[1] = kept;
      if (sweeps_done >= kMaxSweeps) atomicOr(a.status, 2);
    }
    __syncthreads();
    const int k = (int)s_k[0];
    // U columns normalised (a zero column -> e_kk, as the zip-up's a6)
    for (int idx = tid; idx < k * m; idx += kThreads) {
      const int kk = idx / m, i = idx % m, j = perm[kk];
      const double s2 = sg[j];
      A[(size_t)j * m + i] = (s2 > 0.0) ? A[(size_t)j * m + i] / sqrt(s2) : ((i == kk) ? 1.0 : 0.0);
    }
    __syncthreads();
    double *Cq0 = Cw + a.coff[q], *Cq1 = Cw + a.coff[q + 1];
    for (int idx = tid; idx < m * k; idx += kThreads) {
      const int i = idx / k, kk = idx % k;
      Cq0[idx] = A[(size_t)perm[kk] * m + i];
    }
    // C_{q+1}[kk, (i', a'')] = sum_i U[i, kk] M[i, (i', a'')]
    cta_gemm<kThreads>(k, n, m, [&](int kk, int i) { return A[(size_t)perm[kk] * m + i]; },
                       [&](int i, int col) { return S1[(size_t)i * n + col]; },
                       [&](int kk, int col, double v) { Cq1[(size_t)kk * n + col] = v; }, gsm);
    if (tid == 0) {
      cr[q + 1] = k;
      a.norms[(size_t)b * a.sweeps * 2 * L + cnt] = s_k[1];
      if (!isfinite(s_k[1])) atomicOr(a.status, 1);
    }
    ++cnt;
    __syncthreads();
  };
  // Le[q+1][c', (w', r')] = sum_{(c, i)} C_q[(c, i), c'] X2[(c, i), (w', r')]   (C_q left-orthonormal)
  auto left_env = [&](int q) {
    env_apply_left(a, q, cr[q], Le + a.eoff[q], Xq(q), Oq(q), S1, S2, gsm);
    const int w2 = (a.kind == TRUNCATE) ? 1 : a.orr[q + 1], r2 = a.xr[q + 1], k = cr[q + 1];
    const int rows = cr[q] * a.d[q];
    const double *C = Cw + a.coff[q];
    double *L1 = Le + a.eoff[q + 1];
    const int N = w2 * r2;
    cta_gemm<kThreads>(k, N, rows, [&](int i, int kk) { return C[(size_t)kk * k + i]; },
                       [&](int kk, int j) { return S2[(size_t)kk * N + j]; },
                       [&](int i, int j, double v) { L1[(size_t)i * N + j] = v; }, gsm);
    __syncthreads();
  };
  if (a.ncores == 2) {
    for (int sw = 0; sw < a.sweeps; ++sw) {
      for (int q = 0; q < L - 1; ++q) {           // to the right: the centre moves to q+1
        split(q);
        left_env(q);
      }
      for (int q = L - 2; q >= 0; --q) {          // and back: C_{q+1} <- V_k^T by LQ, centre at q
        split(q);
        move_left(q + 1);
        env_right(a, q + 1, cr[q + 1], cr[q + 2], Cw + a.coff[q + 1], Re + a.eoff[q + 2], Xq(q + 1), Oq(q + 1), S1,
                  S2, Re + a.eoff[q + 1], gsm);
      }
    }
  }
  for (int sw = 0; sw < (a.ncores == 2 ? 0 : a.sweeps); ++sw) {
    for (int q = 0; q < L; ++q) {                 // to the right
      update(q);
      if (q == L - 1) break;
      move_right(q);
      // Le[q+1][c', w', r'] = sum_{c, i} C[c, i, c'] X2[c, i, w', r']   (X2 from Le[q])
      env_apply_left(a, q, cr[q], Le + a.eoff[q], Xq(q), Oq(q), S1, S2, gsm);
      const int w2 = (a.kind == TRUNCATE) ? 1 : a.orr[q + 1], r2 = a.xr[q + 1], k = cr[q + 1];
      const int rows = cr[q] * a.d[q];
      const double *C = Cw + a.coff[q];
      double *L1 = Le + a.eoff[q + 1];
      const int N = w2 * r2;
      cta_gemm<kThreads>(k, N, rows, [&](int i, int kk) { return C[(size_t)kk * k + i]; },
                         [&](int kk, int j) { return S2[(size_t)kk * N + j]; },
                         [&](int i, int j, double v) { L1[(size_t)i * N + j] = v; }, gsm);
      __syncthreads();
    }
    for (int q = L - 1; q >= 0; --q) {            // and back
      update(q);
      if (q == 0) break;
      move_left(q);
      env_right(a, q, cr[q], cr[q + 1], Cw + a.coff[q], Re + a.eoff[q + 1], Xq(q), Oq(q), S1, S2, Re + a.eoff[q], gsm);
    }
  }
  // write back (centre at site 0); bonds may have shrunk where a core could not be orthonormal
  for (int q = tid; q <= L; q += kThreads) a.c_ranks[(size_t)b * (L + 1) + q] = cr[q];
  for (int q = 0; q < L; ++q) {
    const long long n = (long long)cr[q] * a.d[q] * cr[q + 1];
    double *dst = a.c[q] + (size_t)b * a.c_bs[q];
    for (long long i = tid; i < n; i += kThreads) dst[i] = Cw[a.coff[q] + i];
  }
}

}  // namespace cplx

static void var_sizes(const Shape &S, const qtt_trains_t *c, int ncores, long long &member, long long *coff,
                      long long *eoff, long long &e_n, long long &s_n, int &pmax) {
  const int L = S.L;
  coff[0] = 0;
  eoff[0] = 0;
  s_n = 1;
  pmax = 64;
  for (int q = 0; q < L; ++q) {
    const long long cq = c->ranks[q], cq1 = c->ranks[q + 1];
    const long long w = (S.kind == TRUNCATE) ? 1 : S.orr[q], w2 = (S.kind == TRUNCATE) ? 1 : S.orr[q + 1];
    coff[q + 1] = coff[q] + cq * S.d[q] * cq1;
    eoff[q + 1] = eoff[q] + cq * w * S.xr[q];
    s_n = std::max(s_n, cq * w * S.dj[q] * S.xr[q + 1]);
    s_n = std::max(s_n, cq * S.d[q] * w2 * S.xr[q + 1]);
    s_n = std::max(s_n, cq * S.d[q] * cq1 * 2);
    s_n = std::max(s_n, cq * w * S.xr[q]);
    s_n = std::max(s_n, cq1 * S.d[q] * (q + 2 <= L ? (long long)c->ranks[std::min(q + 2, L)] : 1));
    pmax = (int)std::max<long long>(pmax, std::max(cq * S.d[q], cq1 * S.d[q]));
    if (ncores == 2 && q + 1 < L) {            // two-site split of (q, q+1)
      const long long d1 = S.d[q + 1], w3 = (S.kind == TRUNCATE) ? 1 : S.orr[q + 2], c2 = c->ranks[q + 2];
      const long long rc = cq * S.d[q];
      s_n = std::max(s_n, rc * w2 * S.dj[q + 1] * S.xr[q + 2]);
      s_n = std::max(s_n, rc * d1 * w3 * S.xr[q + 2]);
      s_n = std::max(s_n, rc * d1 * c2);
      s_n = std::max(s_n, rc * std::min(rc, d1 * c2));
      pmax = (int)std::max<long long>(pmax, std::max(rc, d1 * c2));
    }
  }
  e_n = eoff[L] + 1;
  member = coff[L] + 2 * e_n + 5 * s_n + 3 * (long long)pmax;
  member = (member + 31) & ~31LL;
}

}  // namespace qtt

using namespace qtt;

extern "C" {

size_t qtt_variational_workspace_bytes_ex(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                          const qtt_trains_t *c, int32_t ncores) {
  Shape S;
  if (!c || (ncores != 1 && ncores != 2) || qtt_zipup_analyse(subscripts, op, x, 0, S) != QTT_OK) return 0;
  long long member, coff[65], eoff[65], e_n, s_n;
  int pmax;
  var_sizes(S, c, ncores, member, coff, eoff, e_n, s_n, pmax);
  return (size_t)S.B * member * 8 + 256;
}

size_t qtt_variational_workspace_bytes(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                       const qtt_trains_t *c) {
  return qtt_variational_workspace_bytes_ex(subscripts, op, x, c, 1);
}

qtt_status_t qtt_variational_ex(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                const qtt_trains_t *seed, const int32_t *seed_ranks, const qtt_trains_t *c,
                                int32_t *c_ranks, int32_t sweeps, int32_t ncores, double eps, int32_t max_rank,
                                double *center_norm2, int32_t *status, void *workspace, size_t workspace_bytes,
                                void *stream) {
  Shape S;
  qtt_status_t st = qtt_zipup_analyse(subscripts, op, x, 0, S);
  if (st != QTT_OK) return st;
  if (!seed || !seed->cores || !seed_ranks || !c || !c->cores || !c->ranks || !c_ranks || !center_norm2 || !status) {
    set_error("NULL argument");
    return QTT_EINVAL;
  }
  if ((x->dtype != QTT_F64) || (op && op->dtype != QTT_F64) || c->dtype != QTT_F64 || seed->dtype != QTT_F64) {
    set_error("qtt_variational: QTT_F64 trains only");
    return QTT_EUNSUPPORTED;
  }
  for (const qtt_trains_t *t : {seed, c}) {
    if (t->n_sites != S.L || t->batch != S.B || t->n_legs != 1) { set_error("seed/output train shape mismatch"); return QTT_ESHAPE; }
    for (int q = 0; q < S.L; ++q)
      if (t->d_out[q] != S.d[q]) { set_error("seed/output digit size mismatch at core %d", q); return QTT_ESHAPE; }
  }
  for (int q = 0; q <= S.L; ++q)
    if (c->ranks[q] < seed->ranks[q]) {
      set_error("output capacity %d at bond %d below the seed's %d", c->ranks[q], q, seed->ranks[q]);
      return QTT_ECAPACITY;
    }
  if (sweeps < 1) { set_error("sweeps < 1"); return QTT_EINVAL; }
  if (ncores != 1 && ncores != 2) { set_error("ncores must be 1 or 2"); return QTT_EUNSUPPORTED; }
  if (ncores == 2 && S.L < 2) { set_error("ncores = 2 needs n_sites >= 2"); return QTT_EINVAL; }
  if (!(eps >= 0.0 && eps < 1.0)) { set_error("eps %g outside [0,1)", eps); return QTT_EINVAL; }
  if (S.L > 64) { set_error("n_sites > 64"); return QTT_EUNSUPPORTED; }
  cplx::VarArgs a;
  memset(&a, 0, sizeof(a));
  long long member;
  int pmax;
  var_sizes(S, c, ncores, member, a.coff, a.eoff, a.e_n, a.s_n, pmax);
  if (!workspace || workspace_bytes < (size_t)S.B * member * 8 + 256) {
    set_error("workspace %zu bytes < required %zu", workspace_bytes, (size_t)S.B * member * 8 + 256);
    return QTT_ECAPACITY;
  }
  a.L = S.L; a.B = S.B; a.kind = S.kind; a.op_batch = op ? op->batch : 1; a.sweeps = sweeps;
  a.ncores = ncores; a.eps = eps; a.max_rank = max_rank; a.pmax = pmax;
  for (int q = 0; q < S.L; ++q) {
    a.d[q] = S.d[q]; a.dj[q] = S.dj[q];
    a.x[q] = (const double *)x->cores[q];
    a.x_bs[q] = (long long)x->ranks[q] * x->d_out[q] * x->ranks[q + 1];
    if (op) {
      a.op[q] = (const double *)op->cores[q];
      a.o_bs[q] = (long long)op->ranks[q] * op->d_out[q] * (op->n_legs == 2 ? op->d_in[q] : 1) * op->ranks[q + 1];
    }
    a.sd[q] = (const double *)seed->cores[q];
    a.sd_bs[q] = (long long)seed->ranks[q] * S.d[q] * seed->ranks[q + 1];
    a.c[q] = (double *)c->cores[q];
    a.c_bs[q] = (long long)c->ranks[q] * S.d[q] * c->ranks[q + 1];
  }
  for (int q = 0; q <= S.L; ++q) { a.xr[q] = S.xr[q]; a.orr[q] = S.orr[q]; a.cap[q] = c->ranks[q]; }
  a.sd_ranks = seed_ranks; a.c_ranks = c_ranks; a.norms = center_norm2; a.status = status;
  a.ws = (double *)workspace;
  a.ws_member = member;
  cudaStream_t s = (cudaStream_t)stream;
  QTT_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int32_t), s));
  cplx::k_variational<<<S.B, kThreads, 0, s>>>(a);
  QTT_CUDA_TRY(cudaGetLastError());
  return QTT_OK;
}

qtt_status_t qtt_variational(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                             const qtt_trains_t *c, int32_t *c_ranks, int32_t sweeps, double *center_norm2,
                             int32_t *status, void *workspace, size_t workspace_bytes, void *stream) {
  return qtt_variational_ex(subscripts, op, x, c, c_ranks, c, c_ranks, sweeps, 1, 0.0, 0, center_norm2, status,
                            workspace, workspace_bytes, stream);
}

}  // extern "C"
