// round.cu -- qtt_round (PAPER.md:710 TensorTrain.truncate).
//
// A right-to-left truncated-SVD sweep is the left-to-right truncate-mode zip-up ("i->i") of
// the mirrored train (site order reversed, bond axes swapped).  Members are mirrored into
// capacity-padded slots (zero bond entries beyond the actual ranks leave the tensor
// unchanged), swept by qtt_zipup on the device, and mirrored back packed at the new ranks.
#include <cuda_runtime.h>
#include <string.h>
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace qtt {

constexpr int kMaxL = 64;

struct MirrorArgs {
  int L, B;
  int d[kMaxL];
  int cap_src[kMaxL + 1];          // source capacities (site order of the source)
  const double *src[kMaxL];        // source cores (batch-strided by capacity slot)
  long long src_bs[kMaxL];
  const int *src_ranks;            // device [B][L+1] actual ranks of the source, or NULL
  double *dst[kMaxL];              // destination cores (site q of dst = site L-1-q of src)
  long long dst_bs[kMaxL];
  int pad;                         // 1: write the full capacity slot (zeros outside); 0: packed
  int *dst_ranks;                  // if !pad: device [B][L+1] ranks written (reversed)
};

// One CTA per (member, destination site).
__global__ void k_mirror(MirrorArgs a) {
  const int b = blockIdx.y, qd = blockIdx.x, qs = a.L - 1 - qd;
  const int L1 = a.L + 1;
  const int rl = a.src_ranks ? a.src_ranks[(size_t)b * L1 + qs] : a.cap_src[qs];
  const int rr = a.src_ranks ? a.src_ranks[(size_t)b * L1 + qs + 1] : a.cap_src[qs + 1];
  const int d = a.d[qs];
  const double *s = a.src[qs] + (size_t)b * a.src_bs[qs];        // packed (rl, d, rr)
  double *t = a.dst[qd] + (size_t)b * a.dst_bs[qd];
  if (a.pad) {
    const int cl = a.cap_src[qs + 1], cr = a.cap_src[qs];        // dst slot (cap_src[qs+1], d, cap_src[qs])
    const long long n = (long long)cl * d * cr;
    for (long long idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const int aa = (int)(idx % cr);                            // dst right index = src left index
      const long long t1 = idx / cr;
      const int i = (int)(t1 % d), ap = (int)(t1 / d);           // dst left index = src right index
      t[idx] = (ap < rr && aa < rl) ? s[((size_t)aa * d + i) * rr + ap] : 0.0;
    }
  } else {
    const long long n = (long long)rr * d * rl;                  // dst packed (rr, d, rl)
    for (long long idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const int aa = (int)(idx % rl);
      const long long t1 = idx / rl;
      const int i = (int)(t1 % d), ap = (int)(t1 / d);
      t[idx] = s[((size_t)aa * d + i) * rr + ap];
    }
    if (threadIdx.x == 0) {
      a.dst_ranks[(size_t)b * L1 + qd + 1] = rl;
      if (qd == 0) a.dst_ranks[(size_t)b * L1] = rr;
    }
  }
}

// delta2 of the mirrored sweep -> site order: out[b*L+q] = mass discarded at bond q+1.
__global__ void k_flip_delta(int B, int L, const double *src, double *dst) {
  const int b = blockIdx.x;
  for (int q = threadIdx.x; q < L; q += blockDim.x)
    dst[(size_t)b * L + q] = (q <= L - 2) ? src[(size_t)b * L + (L - 2 - q)] : 0.0;
}

struct RoundPlan {
  int L, B;
  std::vector<int> d, dm, capx, capm, capz;     // mirrored shapes
  std::vector<long long> mel, zel;              // elements per member per site (mirrored input / zip-up out)
  size_t off_m, off_z, off_zr, off_zd, off_zws, zws_bytes, total;
};

static qtt_status_t plan_round(const qtt_trains_t *x, int32_t max_rank, RoundPlan &P) {
  if (!x || !x->ranks || !x->d_out || !x->cores) { set_error("x is NULL"); return QTT_EINVAL; }
  if (x->n_legs != 1) { set_error("qtt_round: MPS only"); return QTT_EUNSUPPORTED; }
  const int L = x->n_sites;
  if (L < 1 || L > kMaxL) { set_error("n_sites outside [1,%d]", kMaxL); return QTT_EUNSUPPORTED; }
  P.L = L; P.B = x->batch;
  P.d.assign(x->d_out, x->d_out + L);
  P.capx.assign(x->ranks, x->ranks + L + 1);
  P.dm.resize(L); P.capm.resize(L + 1);
  for (int q = 0; q < L; ++q) P.dm[q] = P.d[L - 1 - q];
  for (int q = 0; q <= L; ++q) P.capm[q] = P.capx[L - q];
  // mirrored input train descriptor (pointers filled later) for capacity / workspace queries
  std::vector<void *> nul(L, (void *)1);
  qtt_trains_t m{L, 1, P.B, P.dm.data(), nullptr, P.capm.data(), nul.data()};
  P.capz.resize(L + 1);
  qtt_status_t st = qtt_zipup_capacity("i->i", nullptr, &m, max_rank, P.capz.data());
  if (st != QTT_OK) return st;
  P.mel.resize(L); P.zel.resize(L);
  size_t me = 0, ze = 0;
  for (int q = 0; q < L; ++q) {
    P.mel[q] = (long long)P.capm[q] * P.dm[q] * P.capm[q + 1];
    P.zel[q] = (long long)P.capz[q] * P.dm[q] * P.capz[q + 1];
    me += P.mel[q]; ze += P.zel[q];
  }
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~size_t(255); return o; };
  P.off_m = take(sizeof(double) * me * P.B);
  P.off_z = take(sizeof(double) * ze * P.B);
  P.off_zr = take(sizeof(int) * (L + 1) * P.B);
  P.off_zd = take(sizeof(double) * (L + 1) * P.B);
  std::vector<int> capz_copy(P.capz);
  qtt_trains_t z{L, 1, P.B, P.dm.data(), nullptr, capz_copy.data(), nul.data()};
  P.zws_bytes = qtt_zipup_workspace_bytes("i->i", nullptr, &m, &z);
  if (P.zws_bytes == 0) return QTT_EUNSUPPORTED;
  P.off_zws = take(P.zws_bytes);
  P.total = off;
  return QTT_OK;
}

}  // namespace qtt

using namespace qtt;

extern "C" {

qtt_status_t qtt_round_capacity(const qtt_trains_t *x, int32_t max_rank, int32_t *cap) {
  RoundPlan P;
  qtt_status_t st = plan_round(x, max_rank, P);
  if (st != QTT_OK) return st;
  if (!cap) { set_error("cap is NULL"); return QTT_EINVAL; }
  for (int q = 0; q <= P.L; ++q) cap[q] = P.capz[P.L - q];
  return QTT_OK;
}

size_t qtt_round_workspace_bytes(const qtt_trains_t *x, int32_t max_rank) {
  RoundPlan P;
  if (plan_round(x, max_rank, P) != QTT_OK) return 0;
  return P.total;
}

qtt_status_t qtt_round(const qtt_trains_t *x, const int32_t *x_ranks, double eps, int32_t max_rank,
                       const qtt_trains_t *out, int32_t *out_ranks, double *delta2, double *norm2,
                       int32_t *status, void *workspace, size_t workspace_bytes, void *stream) {
  if ((x && x->dtype != QTT_F64) || (out && out->dtype != QTT_F64)) {
    set_error("qtt_round: dtype must be QTT_F64");
    return QTT_EUNSUPPORTED;
  }
  RoundPlan P;
  qtt_status_t st = plan_round(x, max_rank, P);
  if (st != QTT_OK) return st;
  const int L = P.L;
  if (!out || !out->cores || !out->ranks || out->n_sites != L || out->batch != P.B || out->n_legs != 1 ||
      !out_ranks || !delta2 || !norm2 || !status) {
    set_error("qtt_round: bad output arguments");
    return QTT_EINVAL;
  }
  for (int q = 0; q <= L; ++q)
    if (out->ranks[q] < P.capz[L - q]) { set_error("qtt_round: output capacity too small at bond %d", q); return QTT_ECAPACITY; }
  if (!workspace || workspace_bytes < P.total) { set_error("qtt_round workspace %zu < %zu", workspace_bytes, P.total); return QTT_ECAPACITY; }
  cudaStream_t s = (cudaStream_t)stream;
  char *ws = (char *)workspace;
  double *M = (double *)(ws + P.off_m), *Z = (double *)(ws + P.off_z);
  int *zr = (int *)(ws + P.off_zr);
  double *zd = (double *)(ws + P.off_zd);
  std::vector<void *> mp(L), zp(L);
  {
    size_t om = 0, oz = 0;
    for (int q = 0; q < L; ++q) {
      mp[q] = M + om; om += (size_t)P.mel[q] * P.B;
      zp[q] = Z + oz; oz += (size_t)P.zel[q] * P.B;
    }
  }
  // 1. mirror x into capacity-padded slots
  MirrorArgs ma;
  memset(&ma, 0, sizeof(ma));
  ma.L = L; ma.B = P.B; ma.pad = 1; ma.src_ranks = x_ranks;
  for (int q = 0; q < L; ++q) {
    ma.d[q] = P.d[q];
    ma.src[q] = (const double *)x->cores[q];
    ma.src_bs[q] = (long long)P.capx[q] * P.d[q] * P.capx[q + 1];
    ma.dst[q] = (double *)mp[q];
    ma.dst_bs[q] = P.mel[q];
  }
  for (int q = 0; q <= L; ++q) ma.cap_src[q] = P.capx[q];
  k_mirror<<<dim3(L, P.B), kThreads, 0, s>>>(ma);
  QTT_CUDA_TRY(cudaGetLastError());
  // 2. truncate-mode zip-up of the mirrored train
  qtt_trains_t m{L, 1, P.B, P.dm.data(), nullptr, P.capm.data(), mp.data()};
  qtt_trains_t z{L, 1, P.B, P.dm.data(), nullptr, P.capz.data(), zp.data()};
  st = qtt_zipup("i->i", nullptr, &m, eps, max_rank, 0u, &z, zr, zd, norm2, status, nullptr, ws + P.off_zws,
                 P.zws_bytes, stream);
  if (st != QTT_OK) return st;
  // 3. mirror back, packed at the new ranks
  MirrorArgs mb;
  memset(&mb, 0, sizeof(mb));
  mb.L = L; mb.B = P.B; mb.pad = 0; mb.src_ranks = zr; mb.dst_ranks = out_ranks;
  for (int q = 0; q < L; ++q) {
    mb.d[q] = P.dm[q];
    mb.src[q] = (const double *)zp[q];
    mb.src_bs[q] = P.zel[q];
    mb.dst[q] = (double *)out->cores[q];
    mb.dst_bs[q] = (long long)out->ranks[q] * out->d_out[q] * out->ranks[q + 1];
  }
  for (int q = 0; q <= L; ++q) mb.cap_src[q] = P.capz[q];
  k_mirror<<<dim3(L, P.B), kThreads, 0, s>>>(mb);
  QTT_CUDA_TRY(cudaGetLastError());
  k_flip_delta<<<P.B, 64, 0, s>>>(P.B, L, zd, delta2);
  QTT_CUDA_TRY(cudaGetLastError());
  return QTT_OK;
}

}  // extern "C"
