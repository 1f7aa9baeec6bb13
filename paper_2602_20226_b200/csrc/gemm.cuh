// gemm.cuh -- FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) batched strided GEMM for the site
// contractions of the large-member path (SURVEY.md §8(a) a2 "posed as batched GEMMs on FP64
// DMMA tensor cores", a6 carry G = U_k^T T).
//
//   C[z1,z2] (M x N) = A[z1,z2] (M x K) * B[z1,z2] (K x N)
//
// with arbitrary element strides (the contraction operands are views of cores).  The shapes
// and strides live in device memory (ranks are decided on the device), so the grid is sized
// by capacity and surplus CTAs exit.  A is either K-contiguous (row-major, sak == 1) or
// M-contiguous (sam == 1): a template parameter chosen by the launch site; B is N-contiguous.
//
// CTA tile 128 x 128, K chunks of 16, 3-stage cp.async pipeline (8-byte copies: views need
// not be 16-byte aligned; zero-fill outside the matrix), 8 warps as 4 (M) x 2 (N), warp tile
// 32 x 64 = 4 x 8 DMMA fragments (64 fp64 accumulators per lane).  Shared-memory leading
// dimensions are chosen so every fragment load hits each 8-byte bank pair exactly twice per
// warp (the minimum two wavefronts of a 256-byte request).
//
// TMA = true (measured, not the product's feed -- DESIGN.md section 6): an interior tile (all 128 rows /
// columns inside the matrix, K a multiple of 16) of a view whose contiguous dimension has unit
// stride and whose rows start 16-byte aligned (even leading stride, aligned base) is staged by
// TMA bulk copies (`cp.async.bulk` ... `mbarrier::complete_tx`: one 128-byte or 1 KB row per
// copy into the padded fragment layout, issued by warp 0, one mbarrier per stage); every other
// tile (ragged edges, odd strides -- ranks are decided on the device and need not be even --
// and the transposing K-contiguous B) keeps cp.async.  The decision is per CTA and operand and
// both feeds share the stages and the one __syncthreads per K chunk.  On B200 the row-wise bulk
// copies lose to cp.async (cfg3 314 vs 289 ms per zip-up), so libqtt instantiates TMA = false;
// tests/test_gpu_gemm.py checks both.
#pragma once
#include "common.cuh"

namespace qtt {

struct GemmSpec {
  int M, N, K, nz1, nz2;
  const double *A;
  const double *B;
  double *C;
  long long sam, sak, sbk, sbn, scm, scn;
  long long sa1, sa2, sb1, sb2, sc1, sc2;
  int kchunk;        // > 0: split-K -- batch index z1 takes K range [z1 kchunk, (z1+1) kchunk)
                     // (the caller sets sa1 = kchunk sak, sb1 = kchunk sbk, sc1 = the partial stride)
  int upper;         // 1: C is symmetric, only tiles on or above the diagonal are computed
  int tri;           // 1: A[i][k] = 0 for k > i (K stops at the tile's last row);
                     // 2: B[k][j] = 0 for k > j (K stops at the tile's last column)
};

namespace dgemm {
constexpr int TM = 128, TN = 128, TK = 16, STAGES = 3;
constexpr int LDA_K = TK + 4;      // As[m][k] (A K-contiguous): 20 == 4 mod 16
constexpr int LDA_M = TM + 8;      // As[k][m] (A M-contiguous): 136 == 8 mod 16
constexpr int LDB = TN + 8;        // Bs[k][n]: 136
constexpr int A_STAGE = TM * LDA_K > TK * LDA_M ? TM * LDA_K : TK * LDA_M;   // 2560 doubles
constexpr int B_STAGE = TK * LDB;                                            // 2176 doubles
constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double) + STAGES * sizeof(uint64_t);
}  // namespace dgemm

__device__ __forceinline__ void cp_async8(double *dst, const double *src, bool pred) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(dst);
  const int bytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(saddr), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void dmma_884(double &c0, double &c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// grid: x = tiles_m * tiles_n (capacity), z = nz1cap * nz2cap; block = 256 threads.
// B_KCONTIG: B is K-contiguous (sbk == 1, e.g. the transposed operand of a Gram matrix T T^T).
template <bool A_KCONTIG, bool B_KCONTIG = false, bool TMA = false>
__global__ void __launch_bounds__(256, 1) k_gemm_dmma(const GemmSpec *spec, int tiles_n, int nz2_cap) {
  using namespace dgemm;
  extern __shared__ double gsm[];
  GemmSpec g = *spec;
  if (g.kchunk > 0) g.K = min(g.kchunk, g.K - (int)(blockIdx.z / nz2_cap) * g.kchunk);
  if (g.K <= 0) {                                   // empty K chunk: a zero partial
    const int z1 = blockIdx.z / nz2_cap, z2 = blockIdx.z % nz2_cap;
    if (z1 >= g.nz1 || z2 >= g.nz2) return;
    const int m0 = (blockIdx.x / tiles_n) * TM, n0 = (blockIdx.x % tiles_n) * TN;
    double *C = g.C + z1 * g.sc1 + z2 * g.sc2;
    for (int idx = threadIdx.x; idx < TM * TN; idx += 256) {
      const int gm = m0 + idx / TN, gn = n0 + idx % TN;
      if (gm < g.M && gn < g.N) C[(long long)gm * g.scm + (long long)gn * g.scn] = 0.0;
    }
    return;
  }
  const int z1 = blockIdx.z / nz2_cap, z2 = blockIdx.z % nz2_cap;
  if (z1 >= g.nz1 || z2 >= g.nz2) return;
  const int m0 = (blockIdx.x / tiles_n) * TM, n0 = (blockIdx.x % tiles_n) * TN;
  if (m0 >= g.M || n0 >= g.N) return;
  if (g.upper && m0 > n0) return;
  if (g.tri == 1) g.K = min(g.K, m0 + TM);
  if (g.tri == 2) g.K = min(g.K, n0 + TN);
  const double *A = g.A + z1 * g.sa1 + z2 * g.sa2;
  const double *B = g.B + z1 * g.sb1 + z2 * g.sb2;
  double *C = g.C + z1 * g.sc1 + z2 * g.sc2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;          // 4 x 2 warps
  const int gr = lane >> 2, gc = lane & 3;
  double *As = gsm, *Bs = gsm + STAGES * A_STAGE;
  const int nk = (g.K + TK - 1) / TK;

  // TMA feed of interior, 16-byte aligned tiles (CTA-uniform decisions)
  uint64_t *bars = reinterpret_cast<uint64_t *>(gsm + STAGES * (A_STAGE + B_STAGE));
  const bool kfull = TMA && (g.K % TK) == 0;
  const bool tmaA = kfull && m0 + TM <= g.M && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                    (A_KCONTIG ? (g.sam & 1) == 0 : (g.sam == 1 && (g.sak & 1) == 0));
  const bool tmaB = kfull && !B_KCONTIG && n0 + TN <= g.N && (reinterpret_cast<uintptr_t>(B) & 15) == 0 &&
                    g.sbn == 1 && (g.sbk & 1) == 0;
  if (tmaA || tmaB) {
    if (tid == 0)
      for (int st = 0; st < STAGES; ++st) tma_mbar_init(&bars[st]);
    __syncthreads();
  }

  auto load_stage = [&](int st, int kc) {
    const int k0 = kc * TK;
    double *as = As + st * A_STAGE, *bs = Bs + st * B_STAGE;
    if ((tmaA || tmaB) && warp == 0) {
      if (lane == 0)
        tma_expect_tx(&bars[st], (uint32_t)((tmaA ? TM * TK : 0) + (tmaB ? TK * TN : 0)) * (uint32_t)sizeof(double));
      __syncwarp();
      if (tmaA) {
        if (A_KCONTIG) {      // As[m][k]: 128 rows of 16 doubles
#pragma unroll
          for (int e = 0; e < TM / 32; ++e) {
            const int m = e * 32 + lane;
            tma_load_1d(as + m * LDA_K, A + (long long)(m0 + m) * g.sam + k0, TK * sizeof(double), &bars[st]);
          }
        } else if (lane < TK) {   // As[k][m]: 16 rows of 128 doubles
          tma_load_1d(as + lane * LDA_M, A + (long long)(k0 + lane) * g.sak + m0, TM * sizeof(double), &bars[st]);
        }
      }
      if (tmaB && lane >= 32 - TK) {   // Bs[k][n]: 16 rows of 128 doubles
        const int k = lane - (32 - TK);
        tma_load_1d(bs + k * LDB, B + (long long)(k0 + k) * g.sbk + n0, TN * sizeof(double), &bars[st]);
      }
    }
    if (tmaA) {
    } else if (A_KCONTIG) {   // As[m][k]: thread -> row m = tid/2, 8 consecutive k
      const int m = tid >> 1, kh = (tid & 1) * 8, gm = m0 + m;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int gk = k0 + kh + e;
        const bool ok = gm < g.M && gk < g.K;
        cp_async8(as + m * LDA_K + kh + e, ok ? A + (long long)gm * g.sam + gk : A, ok);
      }
    } else {                  // As[k][m]: thread -> k = tid/16, 8 consecutive m
      const int k = tid >> 4, mh = (tid & 15) * 8, gk = k0 + k;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int gm = m0 + mh + e;
        const bool ok = gm < g.M && gk < g.K;
        cp_async8(as + k * LDA_M + mh + e, ok ? A + (long long)gm * g.sam + (long long)gk * g.sak : A, ok);
      }
    }
    if (tmaB) {
    } else if (B_KCONTIG) {   // Bs[k][n] from K-contiguous B: thread -> n = tid/2, 8 consecutive k
      const int n = tid >> 1, kh = (tid & 1) * 8, gn = n0 + n;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int gk = k0 + kh + e;
        const bool ok = gn < g.N && gk < g.K;
        cp_async8(bs + (kh + e) * LDB + n, ok ? B + (long long)gn * g.sbn + gk : B, ok);
      }
    } else {                  // Bs[k][n]: thread -> k = tid/16, 8 consecutive n
      const int k = tid >> 4, nh = (tid & 15) * 8, gk = k0 + k;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int gn = n0 + nh + e;
        const bool ok = gn < g.N && gk < g.K;
        cp_async8(bs + k * LDB + nh + e, ok ? B + (long long)gk * g.sbk + (long long)gn * g.sbn : B, ok);
      }
    }
  };

  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nk) load_stage(st, st);
    cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<STAGES - 2>();
    if (tmaA || tmaB) tma_wait(&bars[kc % STAGES], (uint32_t)(kc / STAGES) & 1u);
    __syncthreads();                                   // stage kc visible; stage kc-1 consumed
    if (kc + STAGES - 1 < nk) load_stage((kc + STAGES - 1) % STAGES, kc + STAGES - 1);
    cp_async_commit();
    const double *as = As + (kc % STAGES) * A_STAGE, *bs = Bs + (kc % STAGES) * B_STAGE;
#pragma unroll
    for (int ks = 0; ks < TK / 4; ++ks) {
      double af[4], bf[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm * 32 + i * 8 + gr, k = ks * 4 + gc;
        af[i] = A_KCONTIG ? as[m * LDA_K + k] : as[k * LDA_M + m];
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) bf[j] = bs[(ks * 4 + gc) * LDB + wn * 64 + j * 8 + gr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  // epilogue: a lane's two adjacent outputs as one 16-byte store when C is N-contiguous and
  // aligned (two 8-byte stores from separate instructions leave every 32-byte sector half
  // written in between: partial-sector writes in L2)
  const bool vec = g.scn == 1 && (g.scm & 1) == 0 && (reinterpret_cast<uintptr_t>(C) & 15) == 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + wm * 32 + i * 8 + gr;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int gn = n0 + wn * 64 + j * 8 + 2 * gc;
      if (vec && gn + 1 < g.N) {
        *reinterpret_cast<double2 *>(C + (long long)gm * g.scm + gn) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e)
          if (gn + e < g.N) C[(long long)gm * g.scm + (long long)(gn + e) * g.scn] = acc[i][j][e];
      }
    }
  }
}

}  // namespace qtt
