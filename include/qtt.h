/* qtt.h -- C-ABI of the B200 zip-up library (libqtt.so).
 *
 * Hot path of arXiv 2602.20226 ("trainsum"): the decomposition / zip-up algorithm of
 * PAPER.md §3.2 (lines 253-275) applying an einsum-style linear map to a quantics tensor
 * train and truncating ranks while it sweeps, plus the exact operations it is checked with
 * (Eq. einsum, inner products SPEC.md:241-249, dense conversion
 * SPEC.md:211-219).  The paper's context-manager options become
 * explicit arguments (eps = ``cutoff``, max_rank), as SPEC.md:416 prescribes.
 *
 * Conventions (all entry points):
 *   - Every core / result pointer is a DEVICE pointer owned by the caller.  The library
 *     never allocates on the hot path (all scratch comes from the caller's workspace) and
 *     never frees caller memory.  Inputs are never modified.
 *   - Layout: MPS core q is row-major (r_q, d_q, r_{q+1}); MPO core q is row-major
 *     (w_q, d_out_q, d_in_q, w_{q+1}).  Digits are big-endian: core 0 holds
 *     the most significant digit (Eq. quantization).
 *   - Batches: a qtt_trains_t describes `batch` members with identical shapes; member b's
 *     core q starts at cores[q] + b * core_elems(q) elements, where
 *     core_elems(q) = ranks[q] * d_out[q] * (d_in[q] if n_legs == 2) * ranks[q+1].
 *     For OUTPUT trains `ranks` are the bond CAPACITIES; every member's core is written
 *     packed at its actual ranks inside its capacity-sized slot.
 *   - dtype: IEEE float64 (the paper's precision) unless a train says otherwise
 *     (qtt_trains_t.dtype: the fp32 and complex128 variants of qtt_zipup).
 *   - Calls are stream-ordered on `stream` (a cudaStream_t passed as void*), asynchronous
 *     (no host synchronisation) and reentrant; there is no global mutable state except
 *     the thread-local error string.
 *   - Errors: a non-QTT_OK status leaves outputs unspecified; qtt_last_error() gives a
 *     human-readable reason for the calling thread.  Numerical failures detected on the
 *     device (non-finite input, Jacobi non-convergence) are reported through the
 *     `status` device word of qtt_zipup (0 = ok) because the call does not synchronise.
 */
#ifndef QTT_H_
#define QTT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QTT_OK = 0,
  QTT_EINVAL = 1,        /* bad argument (NULL pointer, eps outside [0,1), ...)          */
  QTT_ESHAPE = 2,        /* rank chain or extent mismatch                   */
  QTT_ECONFORM = 3,      /* operands do not conform for the subscripts */
  QTT_ENUMERIC = 4,      /* non-finite values / no convergence              */
  QTT_ECAPACITY = 5,     /* output capacity or workspace too small                        */
  QTT_EGUARD = 6,        /* dense size refused                          */
  QTT_ECUDA = 7,         /* CUDA runtime error                                            */
  QTT_EUNSUPPORTED = 8   /* subscript pattern or size not supported by this build         */
} qtt_status_t;

typedef struct {
  int32_t n_sites;        /* L >= 1                                                       */
  int32_t n_legs;         /* 1: MPS core (r, d, r');  2: MPO core (w, d_out, d_in, w')     */
  int32_t batch;          /* B >= 1 members of identical shape                             */
  const int32_t *d_out;   /* host [L] digit sizes (the b_q of Eq. quantization)            */
  const int32_t *d_in;    /* host [L] input digit sizes (MPO) or NULL                       */
  const int32_t *ranks;   /* host [L+1] bond dims (inputs) / bond capacities (outputs);
                             ranks[0] == ranks[L] == 1                                     */
  void *const *cores;     /* host [L] device pointers, batch-strided as described above    */
  int32_t dtype;          /* element type of the cores: QTT_F64 (0, default), QTT_F32 (1) or
                             QTT_C128 (2: complex double, interleaved re/im); QTT_F32 and
                             QTT_C128 are accepted by qtt_zipup only (see there)            */
} qtt_trains_t;

enum { QTT_F64 = 0, QTT_F32 = 1, QTT_C128 = 2 };

/* Flags for qtt_zipup. */
enum {
  QTT_NO_OPERATOR_ORTH = 1u << 0, /* do not right-orthonormalise the operator (SURVEY c-A2) */
  QTT_WINDOW2 = 1u << 1           /* super-core of N = 2 sites:
                                     site q's split is (chi d_q) x (d_{q+1} w_{q+2} r_{q+2}), its
                                     rank capped at w_{q+1} r_{q+1} (the exact product's bond,
                                     reading c-A35); the last split leaves C_{L-1} = diag(s) V^H.
                                     Runs on the per-member path (one CTA per member)          */
};

/* ---------------------------------------------------------------------------------------
 * qtt_zipup_capacity -- output bond capacities for qtt_zipup (host only, no GPU work).
 *   cap[0] = 1; cap[q+1] = min(cap[q]*d_q, w_{q+1}*r_{q+1}, max_rank>0 ? max_rank : inf);
 *   cap[L] = 1.  (The zip-up rank after site q is k <= min(m, n) of its site matrix.)
 *   cap: host [L+1].
 */
qtt_status_t qtt_zipup_capacity(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                int32_t max_rank, int32_t *cap);

/* qtt_zipup_workspace_bytes -- device scratch needed by qtt_zipup for these shapes (flags 0);
 * qtt_zipup_workspace_bytes_flags -- the same for the given qtt_zipup flags (QTT_WINDOW2
 * needs the larger window-2 super-cores).  0 on error (qtt_last_error). */
size_t qtt_zipup_workspace_bytes(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                 const qtt_trains_t *out);
size_t qtt_zipup_workspace_bytes_flags(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                       const qtt_trains_t *out, uint32_t flags);

/* ---------------------------------------------------------------------------------------
 * qtt_zipup -- y = op(x) truncated by the zip-up sweep (window N = 1).
 *
 *   subscripts : "ij,j->i"  op is an MPO (w, d_out, d_in, w'), x an MPS   (matrix-vector)
 *                "i,i->i"   op is an MPS of the same digit shape as x      (Hadamard)
 *                "i->i"     op must be NULL: pure truncation of x (PAPER.md:710 truncate)
 *   Steps per member:
 *     a1 right-orthonormalise every operand by Householder QR;
 *     for q = 0..L-1:
 *       a2 T_q[(chi,i),(w',r')] = sum_{w,r,j} G[chi,w,r] x_q[r,j,r'] op_q[w,i,j,w']
 *          (Hadamard: j == i and op_q[w,i,i,w'] := a_q[w,i,w'])  (Eq. einsum);
 *       a3 R = QR(T^H) when m <= n, else T itself;
 *       a4 one-sided Jacobi SVD -> sigma (descending), U;
 *       a5 k = min(max_rank, smallest k>=1 with sqrt(sum_{j>k} s_j^2) <= eps*||s||)
 *          (SPEC.md:299), delta2_q = sum_{j>k} s_j^2;
 *       a6 C_q = U[:, :k] (chi, d, k);  G <- U_k^T T_q;
 *       a7 last site: C_{L-1} = T_{L-1};  norm2 = ||C_{L-1}||_F^2.
 *   eps        : relative cutoff in [0, 1).       max_rank: <= 0 means unbounded.
 *   out        : output trains, n_legs = 1, ranks[] = capacities (>= qtt_zipup_capacity).
 *   out_ranks  : device int32 [B*(L+1)] actual ranks per member (written).
 *   delta2     : device f64 [B*L]: discarded sum of squares of split q (last entry 0).
 *   norm2      : device f64 [B]: ||y_b||_F^2.
 *   diag       : optional diagnostics (NULL for none), see qtt_zipup_diag_t.
 *   status     : device int32 [1]: 0 on success; bit 1 = non-finite value seen,
 *                bit 2 = Jacobi did not converge (the host status cannot know: no sync).
 *   workspace  : device scratch of >= qtt_zipup_workspace_bytes bytes, 256-byte aligned.
 *   fp32 variant (BASELINE.json configs[2] "fp64 and fp32", c-A27/A28):
 *                when x, op and out all have dtype QTT_F32 the cores are IEEE binary32.  They
 *                are widened into the workspace; the site contractions that run as large
 *                GEMMs (large-member path: state GEMM, Hadamard apply, carry) execute as
 *                3xTF32 on the 5th-generation tensor cores (tcgen05 kind::tf32, fp32
 *                accumulation); QR, Jacobi SVD and truncation run in fp64; the output cores
 *                are rounded to binary32.  Mixed dtypes return QTT_EINVAL.  Accuracy target:
 *                relative Frobenius error <= 1e-4 + eps against the fp64 oracle (c-A28).
 *   complex128 (the tensorized Fourier transform of PAPER.md:533-566 as a
 *                chain of Hadamard zip-ups): when x, op and out all have dtype QTT_C128 the
 *                cores are complex doubles (interleaved re, im; 16 bytes).  Same steps in
 *                complex arithmetic (T^H is the conjugate transpose, the carry is U_k^H T, the
 *                Jacobi rotations carry the phase of a_i^H a_j); delta2, norm2 and sigma stay
 *                real f64.  One CTA per member (complex.cu); diag->phase_cycles gets a2, a3,
 *                a4, a5+a6 per site as for fp64, with the a1 pre-pass in slot [site 0][3].
 */
typedef struct {
  double *sigma;          /* device f64 [B*(L-1)*sigma_stride]: singular values of every site
                             matrix, descending, zero padded; NULL to skip                    */
  int32_t sigma_stride;
  int32_t *sweeps;        /* device int32 [B*L]: Jacobi sweeps run at every site; NULL to skip */
  void *const *events;    /* host [4] cudaEvent_t recorded on `stream`: events[0]/[1] bracket
                             the a1 pre-pass kernels, events[2]/[3] the persistent sweep
                             kernel (a2..a7 for every site and member); NULL to skip (used by
                             bench.py to time the dominant kernel)                           */
  int64_t *phase_cycles;  /* device int64 [B*L*4]: SM clock cycles of the site kernel phases
                             (a2 contraction, a3 QR, a4 Jacobi, a5+a6 truncation/emit/carry)
                             for every member and site; NULL to skip                          */
} qtt_zipup_diag_t;

qtt_status_t qtt_zipup(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                       double eps, int32_t max_rank, uint32_t flags, const qtt_trains_t *out,
                       int32_t *out_ranks, double *delta2, double *norm2, int32_t *status,
                       const qtt_zipup_diag_t *diag, void *workspace, size_t workspace_bytes,
                       void *stream);

/* ---------------------------------------------------------------------------------------
 * qtt_round -- rounding / truncation of a train (PAPER.md:710 ``TensorTrain.truncate``;
 * SURVEY.md §8(f) f1): a right-to-left truncated-SVD sweep with the SPEC.md:299 rule, run
 * as the truncate-mode zip-up ("i->i") of the mirrored train (site order reversed, bond
 * axes swapped), then mirrored back.  Applied to a zip-up output (left-canonical) it is the
 * classical TT rounding and reaches the minimal ranks.
 *   x          : input trains (n_legs 1); x->ranks are capacities; x_ranks (device int32
 *                [B*(L+1)]) gives each member's actual ranks (cores packed inside the
 *                capacity slots, as qtt_zipup writes them); NULL = packed at x->ranks.
 *   out        : output trains; out->ranks are capacities >= qtt_round_capacity.
 *   out_ranks, delta2 (per split, right-to-left order reversed back to site order: delta2[b*L+q]
 *                is the mass discarded at bond q+1), norm2, status: as for qtt_zipup.
 */
qtt_status_t qtt_round_capacity(const qtt_trains_t *x, int32_t max_rank, int32_t *cap);
size_t qtt_round_workspace_bytes(const qtt_trains_t *x, int32_t max_rank);
qtt_status_t qtt_round(const qtt_trains_t *x, const int32_t *x_ranks, double eps, int32_t max_rank,
                       const qtt_trains_t *out, int32_t *out_ranks, double *delta2, double *norm2,
                       int32_t *status, void *workspace, size_t workspace_bytes, void *stream);

/* ---------------------------------------------------------------------------------------
 * qtt_variational -- variational refinement of a zip-up result (Eq.
 * variational 294): minimise |C - op(x)| core by core, single-site,
 * with C(i_q) = d<C|op(x)>/dC*(i_q) at the normalisation centre (reading c-A36).  The seed C
 * is right-orthonormalised (centre at site 0), then `sweeps` times: update sites 0..L-1
 * moving the centre right by QR, then L-1..0 moving it left by LQ.  Bond ranks are the
 * seed's (a bond shrinks only where a core cannot be orthonormal).  QTT_F64 only.
 *   subscripts, op, x : as for qtt_zipup (the operands are not modified, not normalised).
 *   c          : in/out trains (capacity slots as qtt_zipup writes them); on return member b
 *                holds C with the centre at site 0, packed at c_ranks.
 *   c_ranks    : device int32 [B*(L+1)] in: the seed's ranks (qtt_zipup's out_ranks); out: final.
 *   center_norm2 : device f64 [B * sweeps * 2L]: |C_q|^2 after every update, in update order;
 *                |op(x) - C|^2 = |op(x)|^2 - |C_q|^2, so the sequence never decreases.
 *   status     : device int32 [1]; bit 1 = non-finite value.
 *   workspace  : >= qtt_variational_workspace_bytes(subscripts, op, x, c) bytes.
 */
size_t qtt_variational_workspace_bytes(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                       const qtt_trains_t *c);
qtt_status_t qtt_variational(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                             const qtt_trains_t *c, int32_t *c_ranks, int32_t sweeps, double *center_norm2,
                             int32_t *status, void *workspace, size_t workspace_bytes, void *stream);

/* qtt_variational_ex -- the same refinement with multi-core super-cores (PAPER.md:300:
 * "By fusing multiple adjacent C(i_q) into a super-core ... it is possible to realize multi-core
 * strategies, which normally leads to better convergence and an efficient way of controlling
 * the ranks"; the paper's call variational(max_rank=8, cutoff=0.0, ncores=2, nsweeps=2),
 * PAPER.md:794; reading c-A37).
 *   seed, seed_ranks : the starting train (device int32 [B*(L+1)] ranks); read completely
 *                before anything is written, so it may alias c / c_ranks.
 *   c, c_ranks : output slots (capacities c->ranks >= seed->ranks; with ncores = 2 the bond
 *                ranks adapt up to min(max_rank, capacity)), final ranks written to c_ranks;
 *                on return the centre is at site 0 (cores 1..L-1 right-orthonormal).
 *   ncores     : 1 (as qtt_variational) or 2: the super-core of sites (q, q+1),
 *                S = Le[q] W_q x_q W_{q+1} x_{q+1} Re[q+2], is split by Householder QR + one-sided
 *                Jacobi and truncated by the zip-up's rule (SPEC.md:299 with eps = cutoff,
 *                k <= max_rank (<= 0: unbounded), k <= capacity); a sweep updates the pairs
 *                q = 0..L-2 (centre moving right) then L-2..0 (an LQ moves it left).
 *   center_norm2 : device f64 [B * sweeps * 2L]; ncores = 2 writes 2(L-1) values per sweep,
 *                the kept |S_k|^2 = sum_{j<=k} s_j^2 of each split.
 *   workspace  : >= qtt_variational_workspace_bytes_ex(subscripts, op, x, c, ncores) bytes.
 * Errors: QTT_ECAPACITY (capacity below the seed's ranks or workspace), QTT_ESHAPE, QTT_EINVAL
 * (eps outside [0,1), sweeps < 1, ncores = 2 with one site), QTT_EUNSUPPORTED (ncores not 1/2,
 * non-f64 trains).  status bit 1 = non-finite value, bit 2 = Jacobi did not converge. */
size_t qtt_variational_workspace_bytes_ex(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                          const qtt_trains_t *c, int32_t ncores);
qtt_status_t qtt_variational_ex(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                const qtt_trains_t *seed, const int32_t *seed_ranks, const qtt_trains_t *c,
                                int32_t *c_ranks, int32_t sweeps, int32_t ncores, double eps, int32_t max_rank,
                                double *center_norm2, int32_t *status, void *workspace, size_t workspace_bytes,
                                void *stream);

/* ---------------------------------------------------------------------------------------
 * qtt_zipup_sharded -- ONE zip-up (fp64, batch 1, large-member path) split across the
 * processes of a job, one GPU each (SURVEY.md §8(f) f4 "cross-GPU sharding of one zip-up",
 * §8(e); the site matrix T_q -- "contracted exactly" -- is split by the
 * SVD of PAPER.md:257/269).  The columns of every site matrix T_q (m = chi d rows, columns
 * (w', r')) are split into S = world * local_shards shards by contiguous, balanced ranges of
 * the state bond r' (r_{q+1}); shard t = rank * local_shards + s.  Per site:
 *   1. each process contracts its shards' column slabs T_t = contract(G, x_q[:, :, r'-slice],
 *      op_q) from the full carry G, and reduces each to an m x m factor F_t with
 *      F_t^T F_t = T_t T_t^T (the R of T_t^H by the Householder QR of a3 when the slab has at
 *      least m columns, else T_t^H itself), zero-padded to mcap x mcap, into send_r;
 *   2. allgather(0): recv_r[t] = every shard's F_t (all processes, shard order);
 *   3. R = the R of the stacked [F_0; ...; F_{S-1}] (same QR) -- the R of T^H, since
 *      T T^T = sum_t F_t^T F_t; then a4-a6 exactly as qtt_zipup: one-sided Jacobi on R^T,
 *      the SPEC.md:299 truncation (k <= min(max_rank, w' r')), C_q = U_k written by every
 *      process (identical values on all);
 *   4. each process forms its carry slabs U_k^T T_t (k x w' x slice) into send_c;
 *   5. allgather(1): recv_c[t] = every shard's carry slab; the full carry (k, w', r') is
 *      assembled for the next site.
 * The last site (n = 1) and a1 run unsharded on every process.  Exchanges per site: S
 * mcap^2 + S kcap ncap_slab doubles (the carry all-gather is the "carry exchange").
 *   comm->allgather(phase, user) must ENQUEUE the all-gather of the phase's buffers on the
 *   stream (e.g. torch.distributed / NCCL on the current stream) and return 0; it is called
 *   from this function, in site order, the same number of times on every process.  With
 *   world == 1 it may be NULL: the library copies send -> recv itself (several shards in one
 *   process -- the same arithmetic as S processes).
 *   Buffer sizes: qtt_zipup_sharded_sizes() -> elements of ONE shard's R slab and carry slab;
 *   send_* hold local_shards slabs, recv_* hold world * local_shards.
 * Outputs as qtt_zipup (member 0).  Errors: QTT_EUNSUPPORTED for batch != 1, non-f64,
 * QTT_WINDOW2 or a site matrix the large-member path cannot stage; QTT_EINVAL for a bad comm.
 */
typedef int (*qtt_allgather_fn)(int32_t phase, void *user);
typedef struct {
  int32_t world, rank, local_shards;
  qtt_allgather_fn allgather;
  void *user;
  double *send_r, *recv_r;   /* device: [local_shards] / [world*local_shards] x r_elems  */
  double *send_c, *recv_c;   /* device: [local_shards] / [world*local_shards] x c_elems  */
} qtt_shard_comm_t;
qtt_status_t qtt_zipup_sharded_sizes(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x,
                                     int32_t max_rank, int32_t world, int32_t local_shards, size_t *r_elems,
                                     size_t *c_elems, size_t *workspace_bytes);
qtt_status_t qtt_zipup_sharded(const char *subscripts, const qtt_trains_t *op, const qtt_trains_t *x, double eps,
                               int32_t max_rank, uint32_t flags, const qtt_trains_t *out, int32_t *out_ranks,
                               double *delta2, double *norm2, int32_t *status, double *sigma, int32_t sigma_stride,
                               const qtt_shard_comm_t *comm, void *workspace, size_t workspace_bytes,
                               void *stream);

/* qtt_zipup_summary -- the per-batch scalars that are all-reduced across GPUs
 * (SURVEY.md §8(a) a8): summary4 (device f64 [4]) = [sum_b sum_q delta2, sum_b norm2,
 * sum_b sum_q out_ranks[b][q+1] (q < L-1), B].  Deterministic fixed-order sums. */
qtt_status_t qtt_zipup_summary(int32_t batch, int32_t n_sites, const int32_t *out_ranks,
                               const double *delta2, const double *norm2, double *summary4, void *stream);

/* ---------------------------------------------------------------------------------------
 * qtt_einsum_exact -- exact einsum by local summation (Eq. einsum):
 *   "ij,j->i": C_q[(w,r), i, (w',r')] = sum_j a_q[w,i,j,w'] b_q[r,j,r']
 *   "i,i->i" : C_q[(a,b), i, (a',b')] = a_q[a,i,a'] b_q[b,i,b']
 * Bond indices are flattened first-operand-slow (xi = mu nu).  out->ranks must equal the
 * products of the operand ranks; out->n_legs = 1.
 */
qtt_status_t qtt_einsum_exact(const char *subscripts, const qtt_trains_t *a, const qtt_trains_t *b,
                              const qtt_trains_t *out, void *stream);

/* qtt_inner -- <a, b> for every member (left-to-right environments);
 * a and b must be addition-compatible (same n_legs and digit sizes).  result: device
 * f64 [B].  workspace: >= qtt_inner_workspace_bytes(a, b). */
size_t qtt_inner_workspace_bytes(const qtt_trains_t *a, const qtt_trains_t *b);
qtt_status_t qtt_inner(const qtt_trains_t *a, const qtt_trains_t *b, double *result,
                       void *workspace, size_t workspace_bytes, void *stream);

/* qtt_to_dense -- dense tensor of every member, row-major over the
 * original (unfactorised) dimensions: leg_dim[q] (host [L], or NULL = all one dimension)
 * names the dimension of site q's digit; digits of one dimension appear in order, most
 * significant first.  MPS only.  out: device f64 [B * prod(d)].  Refuses with QTT_EGUARD
 * when prod(d) > max_elems (inclusive guard; max_elems <= 0 means 2^24, SURVEY c-A30). */
size_t qtt_to_dense_workspace_bytes(const qtt_trains_t *t);
qtt_status_t qtt_to_dense(const qtt_trains_t *t, const int32_t *leg_dim, double *out, int64_t max_elems,
                          void *workspace, size_t workspace_bytes, void *stream);

/* Thread-local description of the last error on this thread ("" if none). */
const char *qtt_last_error(void);

/* Library version string. */
const char *qtt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QTT_H_ */
