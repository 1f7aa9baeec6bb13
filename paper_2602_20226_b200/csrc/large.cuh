// large.cuh -- shared declarations between zipup.cu (small-member path, host entry) and
// large.cu (large-member path for site matrices with m > 128 rows).
#pragma once
#include <vector>
#include "common.cuh"

namespace qtt {

enum Kind { MATVEC = 0, HADAMARD = 1, TRUNCATE = 2 };
enum StatusBits { ST_NONFINITE = 1, ST_NOCONV = 2 };

struct Shape {
  int L = 0, B = 0, kind = 0, shared_op = 0;
  std::vector<int> d, dj, xr, orr, cap;
  std::vector<long long> xoff, ooff;
  long long xo_elems = 0, oo_elems = 0, g_elems = 1, t_elems = 1, x_elems = 1;
};

// Large-member path entry (large.cu).  Operands are already copied into Xo / Oo (capacity
// slots, batch-strided) with device ranks xr / orr, and right-orthonormalised unless
// `skip_orth` asks the large path to do it (mirrored truncate sweeps).
struct LargeIO {
  const qtt_trains_t *out;
  int32_t *out_ranks;
  double *delta2, *norm2, *sigma;
  int sigma_stride;
  int *sweeps;
  int *status;
  double eps;
  int max_rank;
};

size_t large_workspace_bytes(const Shape &S);
// the fp64 a1 pre-pass (zipup.cu k_orth) into caller-given member slots (per-member kernel)
qtt_status_t orth_prepass(const Shape &S, const qtt_trains_t *op, const qtt_trains_t *x, uint32_t flags, double *xdst,
                          double *odst, long long dst_bs, int *xr_out, int *orr_out, cudaStream_t s);
// shape analysis of qtt_zipup's operands (zipup.cu), shared with qtt_variational
qtt_status_t qtt_zipup_analyse(const char *subs, const qtt_trains_t *op, const qtt_trains_t *x, int32_t max_rank,
                               Shape &S);
// per-member path (complex.cu): one CTA per member, every step; complex128 trains (f2) and
// the window-2 zip-up (f4, real or complex)
size_t member_workspace_bytes(const Shape &S, int elem_bytes, int window);
bool a1_fits(const Shape &S, bool report);
qtt_status_t member_zipup(const Shape &S, const qtt_trains_t *op, const qtt_trains_t *x, uint32_t flags,
                          const struct LargeIO &io, void *workspace, size_t workspace_bytes, cudaStream_t s,
                          long long *cycles, bool complex_dt, int window, void *const *events);
qtt_status_t large_zipup(const Shape &S, const qtt_trains_t *op, const qtt_trains_t *x, uint32_t flags,
                         const LargeIO &io, void *workspace, size_t workspace_bytes, cudaStream_t s);

}  // namespace qtt
