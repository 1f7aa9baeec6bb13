// exact.cu -- exact operations used to check and consume the zip-up output:
//   qtt_einsum_exact : Eq. einsum, ranks multiply
//   qtt_inner        : <a,b> by left-to-right environments
//   qtt_to_dense     : dense tensor over the original dimensions
//   qtt_zipup_summary: fixed-order per-batch sums that are all-reduced across GPUs (a8)
#include <cuda_runtime.h>
#include <string.h>
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace qtt {

// ------------------------------------------------------------------ einsum (exact)

__global__ void k_einsum_site(int hadamard, const double *A, long long A_bs, const double *Bc, long long B_bs,
                              double *C, long long C_bs, int ra, int ra2, int rb, int rb2, int di, int dj,
                              long long total) {
  const int b = blockIdx.y;
  const double *Am = A + (size_t)b * A_bs;
  const double *Bm = Bc + (size_t)b * B_bs;
  double *Cm = C + (size_t)b * C_bs;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int col = (int)(idx % ((long long)ra2 * rb2));
    long long t = idx / ((long long)ra2 * rb2);
    const int i = (int)(t % di);
    const int row = (int)(t / di);
    const int wa = row / rb, wb = row % rb, wa2 = col / rb2, wb2 = col % rb2;
    double s;
    if (hadamard) {
      s = Am[((size_t)wa * di + i) * ra2 + wa2] * Bm[((size_t)wb * di + i) * rb2 + wb2];
    } else {
      s = 0.0;
      for (int j = 0; j < dj; ++j)
        s = fma(Am[(((size_t)wa * di + i) * dj + j) * ra2 + wa2], Bm[((size_t)wb * dj + j) * rb2 + wb2], s);
    }
    Cm[idx] = s;
  }
}

// ------------------------------------------------------------------ generic tiled GEMM

// C[b] = A[b] (M x K, lda) * B[b] (K x N, ldb), one 64x64 tile per CTA (grid y = tiles, z = batch).
__global__ void __launch_bounds__(kThreads) k_gemm(int M, int N, int K, const double *A, long long lda, long long A_bs,
                                                   const double *Bm, long long ldb, long long B_bs, double *C,
                                                   long long ldc, long long C_bs) {
  __shared__ double sm[2 * 16 * 64];
  const int b = blockIdx.z;
  const int tiles_n = (N + 63) / 64;
  const int m0 = (blockIdx.x / tiles_n) * 64, n0 = (blockIdx.x % tiles_n) * 64;
  const double *Ab = A + (size_t)b * A_bs + (size_t)m0 * lda;
  const double *Bb = Bm + (size_t)b * B_bs + n0;
  double *Cb = C + (size_t)b * C_bs + (size_t)m0 * ldc + n0;
  const int Mt = min(64, M - m0), Nt = min(64, N - n0);
  cta_gemm(Mt, Nt, K, [&](int i, int k) { return Ab[(size_t)i * lda + k]; },
           [&](int k, int j) { return Bb[(size_t)k * ldb + j]; },
           [&](int i, int j, double v) { Cb[(size_t)i * ldc + j] = v; }, sm);
}

static qtt_status_t launch_gemm(int B, int M, int N, int K, const double *A, long long lda, long long A_bs,
                                const double *Bm, long long ldb, long long B_bs, double *C, long long ldc,
                                long long C_bs, cudaStream_t s) {
  const long long tiles = (long long)((M + 63) / 64) * ((N + 63) / 64);
  if (tiles > 0x7fffffffLL || B > 65535) { set_error("gemm grid too large"); return QTT_EUNSUPPORTED; }
  dim3 grid((unsigned)tiles, 1, (unsigned)B);
  k_gemm<<<grid, kThreads, 0, s>>>(M, N, K, A, lda, A_bs, Bm, ldb, B_bs, C, ldc, C_bs);
  QTT_CUDA_TRY(cudaGetLastError());
  return QTT_OK;
}

// ------------------------------------------------------------------ inner product

// One CTA per member: E <- sum_l A_q[:,l,:]^T E B_q[:,l,:] (two CTA GEMMs per site).
struct InnerArgs {
  int L;
  int legs[64];
  int ra[65], rb[65];
  const double *A[64]; long long Abs[64];
  const double *Bc[64]; long long Bbs[64];
  double *ws; long long ws_bs; long long e_elems;   // E0 | E1 | F per member
  double *result;
};

__global__ void __launch_bounds__(kThreads, 1) k_inner(InnerArgs a) {
  __shared__ double sm[2 * 16 * 64];
  const int b = blockIdx.x;
  double *E = a.ws + (size_t)b * a.ws_bs;
  double *E2 = E + a.e_elems;
  double *F = E2 + a.e_elems;
  if (threadIdx.x == 0) E[0] = 1.0;
  __syncthreads();
  for (int q = 0; q < a.L; ++q) {
    const double *Aq = a.A[q] + (size_t)b * a.Abs[q];
    const double *Bq = a.Bc[q] + (size_t)b * a.Bbs[q];
    const int ra = a.ra[q], rb = a.rb[q], ra2 = a.ra[q + 1], rb2 = a.rb[q + 1], l = a.legs[q];
    // F[bb][(l, c)] = sum_aa E[aa][bb] A[aa][(l,c)]
    cta_gemm(rb, l * ra2, ra, [&](int bb, int aa) { return E[(size_t)aa * rb + bb]; },
             [&](int aa, int lc) { return Aq[(size_t)aa * l * ra2 + lc]; },
             [&](int bb, int lc, double v) { F[(size_t)bb * l * ra2 + lc] = v; }, sm);
    __syncthreads();
    // E2[c][dd] = sum_{bb,ll} F[bb][ll][c] B[bb][ll][dd]
    cta_gemm(ra2, rb2, rb * l, [&](int c, int bl) { return F[(size_t)bl * ra2 + c]; },
             [&](int bl, int dd) { return Bq[(size_t)bl * rb2 + dd]; },
             [&](int c, int dd, double v) { E2[(size_t)c * rb2 + dd] = v; }, sm);
    __syncthreads();
    double *t = E; E = E2; E2 = t;
  }
  if (threadIdx.x == 0) a.result[b] = E[0];
}

// ------------------------------------------------------------------ dense permutation

struct PermArgs {
  int L;
  int d[64];
  long long src_stride[64];   // row-major over sites
  long long dst_stride[64];   // row-major over the dimension-grouped order
};

__global__ void k_permute(PermArgs p, const double *src, long long src_bs, double *dst, long long dst_bs,
                          long long total) {
  const int b = blockIdx.y;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    long long rem = idx, o = 0;
    for (int q = 0; q < p.L; ++q) {
      const long long dig = rem / p.src_stride[q];
      rem -= dig * p.src_stride[q];
      o += dig * p.dst_stride[q];
    }
    dst[(size_t)b * dst_bs + o] = src[(size_t)b * src_bs + idx];
  }
}

// ------------------------------------------------------------------ summary (a8)

__global__ void k_summary(int B, int L, const int *yr, const double *d2, const double *n2, double *out) {
  __shared__ double red[3][kThreads];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (int b = threadIdx.x; b < B; b += kThreads) {
    for (int q = 0; q < L; ++q) s0 += d2[(size_t)b * L + q];
    s1 += n2[b];
    for (int q = 1; q < L; ++q) s2 += (double)yr[(size_t)b * (L + 1) + q];
  }
  red[0][threadIdx.x] = s0; red[1][threadIdx.x] = s1; red[2][threadIdx.x] = s2;
  __syncthreads();
  for (int o = kThreads / 2; o > 0; o >>= 1) {   // fixed-shape tree: deterministic
    if (threadIdx.x < o)
      for (int c = 0; c < 3; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = red[0][0]; out[1] = red[1][0]; out[2] = red[2][0]; out[3] = (double)B; }
}

static long long core_elems(const qtt_trains_t *t, int q) {
  long long e = (long long)t->ranks[q] * t->d_out[q] * t->ranks[q + 1];
  if (t->n_legs == 2) e *= t->d_in[q];
  return e;
}

static qtt_status_t check_train(const qtt_trains_t *t, const char *name) {
  if (t && t->dtype != QTT_F64) { set_error("%s: dtype must be QTT_F64 for this call", name); return QTT_EUNSUPPORTED; }
  if (!t || !t->cores || !t->ranks || !t->d_out) { set_error("%s: NULL train", name); return QTT_EINVAL; }
  if (t->n_sites < 1 || t->n_sites > 64) { set_error("%s: n_sites outside [1,64]", name); return QTT_EUNSUPPORTED; }
  if (t->n_legs != 1 && t->n_legs != 2) { set_error("%s: n_legs must be 1 or 2", name); return QTT_EINVAL; }
  if (t->n_legs == 2 && !t->d_in) { set_error("%s: MPO without d_in", name); return QTT_EINVAL; }
  if (t->ranks[0] != 1 || t->ranks[t->n_sites] != 1) { set_error("%s: boundary ranks must be 1", name); return QTT_ESHAPE; }
  if (t->batch < 1 || t->batch > 65535) { set_error("%s: batch outside [1,65535]", name); return QTT_EINVAL; }
  return QTT_OK;
}

}  // namespace qtt

using namespace qtt;

extern "C" {

qtt_status_t qtt_einsum_exact(const char *subscripts, const qtt_trains_t *a, const qtt_trains_t *b,
                              const qtt_trains_t *out, void *stream) {
  qtt_status_t st;
  if ((st = check_train(a, "a")) != QTT_OK || (st = check_train(b, "b")) != QTT_OK ||
      (st = check_train(out, "out")) != QTT_OK)
    return st;
  int hadamard;
  if (subscripts && strcmp(subscripts, "ij,j->i") == 0) hadamard = 0;
  else if (subscripts && strcmp(subscripts, "i,i->i") == 0) hadamard = 1;
  else { set_error("unsupported subscripts '%s'", subscripts ? subscripts : "(null)"); return QTT_EUNSUPPORTED; }
  const int L = a->n_sites;
  if (b->n_sites != L || out->n_sites != L) { set_error("site count mismatch"); return QTT_ECONFORM; }
  if (a->n_legs != (hadamard ? 1 : 2) || b->n_legs != 1 || out->n_legs != 1) {
    set_error("operand kinds do not match '%s'", subscripts);
    return QTT_ESHAPE;
  }
  if (!(a->batch == b->batch && b->batch == out->batch)) { set_error("batch mismatch"); return QTT_EINVAL; }
  for (int q = 0; q < L; ++q) {
    const int dj = hadamard ? a->d_out[q] : a->d_in[q];
    if (dj != b->d_out[q]) { set_error("conformance: contracted digit misaligned at core %d", q); return QTT_ECONFORM; }
    if (out->d_out[q] != a->d_out[q]) { set_error("output digit size mismatch at core %d", q); return QTT_ESHAPE; }
  }
  for (int q = 0; q <= L; ++q) {
    if (out->ranks[q] != a->ranks[q] * b->ranks[q]) {
      set_error("output rank %d at bond %d must equal %d*%d (SPEC.md:411)", out->ranks[q], q, a->ranks[q], b->ranks[q]);
      return QTT_ESHAPE;
    }
  }
  cudaStream_t s = (cudaStream_t)stream;
  for (int q = 0; q < L; ++q) {
    const long long total = core_elems(out, q);
    const int di = a->d_out[q], dj = hadamard ? di : a->d_in[q];
    dim3 grid((unsigned)std::min<long long>((total + kThreads - 1) / kThreads, 4096), (unsigned)a->batch);
    k_einsum_site<<<grid, kThreads, 0, s>>>(hadamard, (const double *)a->cores[q], core_elems(a, q),
                                            (const double *)b->cores[q], core_elems(b, q), (double *)out->cores[q],
                                            total, a->ranks[q], a->ranks[q + 1], b->ranks[q], b->ranks[q + 1], di, dj,
                                            total);
    QTT_CUDA_TRY(cudaGetLastError());
  }
  return QTT_OK;
}

size_t qtt_inner_workspace_bytes(const qtt_trains_t *a, const qtt_trains_t *b) {
  if (check_train(a, "a") != QTT_OK || check_train(b, "b") != QTT_OK) return 0;
  long long e = 1, f = 1;
  for (int q = 0; q < a->n_sites; ++q) {
    const long long legs = (long long)a->d_out[q] * (a->n_legs == 2 ? a->d_in[q] : 1);
    e = std::max(e, (long long)a->ranks[q + 1] * b->ranks[q + 1]);
    f = std::max(f, (long long)b->ranks[q] * legs * a->ranks[q + 1]);
  }
  e = (e + 3) & ~3LL;
  return sizeof(double) * (size_t)(2 * e + f) * a->batch;
}

qtt_status_t qtt_inner(const qtt_trains_t *a, const qtt_trains_t *b, double *result, void *workspace,
                       size_t workspace_bytes, void *stream) {
  qtt_status_t st;
  if ((st = check_train(a, "a")) != QTT_OK || (st = check_train(b, "b")) != QTT_OK) return st;
  const int L = a->n_sites;
  if (b->n_sites != L || a->n_legs != b->n_legs || a->batch != b->batch) {
    set_error("inner: shapes not addition-compatible");
    return QTT_ESHAPE;
  }
  for (int q = 0; q < L; ++q) {
    if (a->d_out[q] != b->d_out[q] || (a->n_legs == 2 && a->d_in[q] != b->d_in[q])) {
      set_error("inner: digit sizes differ at core %d", q);
      return QTT_ESHAPE;
    }
  }
  if (!result) { set_error("result is NULL"); return QTT_EINVAL; }
  const size_t need = qtt_inner_workspace_bytes(a, b);
  if (!workspace || workspace_bytes < need) { set_error("inner workspace %zu < %zu", workspace_bytes, need); return QTT_ECAPACITY; }
  InnerArgs ia;
  memset(&ia, 0, sizeof(ia));
  ia.L = L;
  long long e = 1, f = 1;
  for (int q = 0; q < L; ++q) {
    ia.legs[q] = a->d_out[q] * (a->n_legs == 2 ? a->d_in[q] : 1);
    ia.A[q] = (const double *)a->cores[q]; ia.Abs[q] = core_elems(a, q);
    ia.Bc[q] = (const double *)b->cores[q]; ia.Bbs[q] = core_elems(b, q);
    e = std::max(e, (long long)a->ranks[q + 1] * b->ranks[q + 1]);
    f = std::max(f, (long long)b->ranks[q] * ia.legs[q] * a->ranks[q + 1]);
  }
  for (int q = 0; q <= L; ++q) { ia.ra[q] = a->ranks[q]; ia.rb[q] = b->ranks[q]; }
  e = (e + 3) & ~3LL;
  ia.e_elems = e;
  ia.ws = (double *)workspace;
  ia.ws_bs = 2 * e + f;
  ia.result = result;
  k_inner<<<a->batch, kThreads, 0, (cudaStream_t)stream>>>(ia);
  QTT_CUDA_TRY(cudaGetLastError());
  return QTT_OK;
}

size_t qtt_to_dense_workspace_bytes(const qtt_trains_t *t) {
  if (check_train(t, "t") != QTT_OK) return 0;
  long long P = 1, mx = 1;
  for (int q = 0; q < t->n_sites; ++q) {
    P *= t->d_out[q];
    mx = std::max(mx, P * t->ranks[q + 1]);
  }
  return sizeof(double) * (size_t)(2 * mx) * t->batch;
}

qtt_status_t qtt_to_dense(const qtt_trains_t *t, const int32_t *leg_dim, double *out, int64_t max_elems,
                          void *workspace, size_t workspace_bytes, void *stream) {
  qtt_status_t st;
  if ((st = check_train(t, "t")) != QTT_OK) return st;
  if (t->n_legs != 1) { set_error("to_dense: MPS only"); return QTT_EUNSUPPORTED; }
  if (!out) { set_error("out is NULL"); return QTT_EINVAL; }
  const int L = t->n_sites;
  long long N = 1;
  for (int q = 0; q < L; ++q) N *= t->d_out[q];
  const long long guard = max_elems > 0 ? max_elems : (1LL << 24);
  if (N > guard) { set_error("dense size %lld exceeds guard %lld (SPEC.md:213-215)", N, guard); return QTT_EGUARD; }
  const size_t need = qtt_to_dense_workspace_bytes(t);
  if (!workspace || workspace_bytes < need) { set_error("to_dense workspace %zu < %zu", workspace_bytes, need); return QTT_ECAPACITY; }
  cudaStream_t s = (cudaStream_t)stream;
  long long mx = 1, P = 1;
  for (int q = 0; q < L; ++q) { P *= t->d_out[q]; mx = std::max(mx, P * t->ranks[q + 1]); }
  double *V0 = (double *)workspace, *V1 = V0 + (size_t)mx * t->batch;
  // V <- core_0 (d_0 x r_1); V <- V (P x r_q) * core_q (r_q x d_q r_{q+1})
  long long e0 = core_elems(t, 0);
  QTT_CUDA_TRY(cudaMemcpy2DAsync(V0, sizeof(double) * mx, t->cores[0], sizeof(double) * e0, sizeof(double) * e0,
                                 t->batch, cudaMemcpyDeviceToDevice, s));
  P = t->d_out[0];
  for (int q = 1; q < L; ++q) {
    const int rq = t->ranks[q], n = t->d_out[q] * t->ranks[q + 1];
    st = launch_gemm(t->batch, (int)P, n, rq, V0, rq, mx, (const double *)t->cores[q], n, core_elems(t, q), V1, n, mx, s);
    if (st != QTT_OK) return st;
    std::swap(V0, V1);
    P *= t->d_out[q];
  }
  // permute site-digit order into dimension order
  PermArgs pa;
  memset(&pa, 0, sizeof(pa));
  pa.L = L;
  std::vector<int> order;
  std::vector<int> dimid(L, 0);
  if (leg_dim) for (int q = 0; q < L; ++q) dimid[q] = leg_dim[q];
  std::vector<int> ids(dimid);
  std::sort(ids.begin(), ids.end());
  ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
  for (int id : ids)
    for (int q = 0; q < L; ++q)
      if (dimid[q] == id) order.push_back(q);
  long long st_src = 1;
  for (int q = L - 1; q >= 0; --q) { pa.src_stride[q] = st_src; st_src *= t->d_out[q]; }
  long long st_dst = 1;
  for (int u = L - 1; u >= 0; --u) { pa.dst_stride[order[u]] = st_dst; st_dst *= t->d_out[order[u]]; }
  dim3 grid((unsigned)std::min<long long>((N + kThreads - 1) / kThreads, 4096), (unsigned)t->batch);
  k_permute<<<grid, kThreads, 0, s>>>(pa, V0, mx, out, N, N);
  QTT_CUDA_TRY(cudaGetLastError());
  return QTT_OK;
}

qtt_status_t qtt_zipup_summary(int32_t batch, int32_t n_sites, const int32_t *out_ranks, const double *delta2,
                               const double *norm2, double *summary4, void *stream) {
  if (batch < 1 || n_sites < 1 || !out_ranks || !delta2 || !norm2 || !summary4) {
    set_error("qtt_zipup_summary: bad arguments");
    return QTT_EINVAL;
  }
  k_summary<<<1, kThreads, 0, (cudaStream_t)stream>>>(batch, n_sites, out_ranks, delta2, norm2, summary4);
  QTT_CUDA_TRY(cudaGetLastError());
  return QTT_OK;
}

}  // extern "C"
