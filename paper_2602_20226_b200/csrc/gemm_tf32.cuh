// gemm_tf32.cuh -- 3xTF32 batched strided GEMM on the 5th-generation tensor cores (tcgen05
// kind::tf32, accumulators in TMEM) for the fp32 variant of the large-member contractions
// (BASELINE.json north_star "(with a TF32/FP32 variant)").
//
//   C[z1,z2] (M x N, fp64 storage) = A[z1,z2] (M x K) * B[z1,z2] (K x N)
//
// Operands are read from fp64 storage, rounded to fp32 and split x = hi + lo with hi, lo
// TF32 (cvt.rna.tf32.f32); the product is hi*hi + hi*lo + lo*hi (the lo*lo term is below
// fp32 resolution), which restores ~fp32 accuracy on the TF32 tensor pipe.  Four fp32 TMEM
// accumulators (hi*hi and the two correction terms kept apart, each split by K-chunk
// parity) are summed in fp64 in the epilogue: the small correction terms are not rounded
// against the large hi*hi partial sums, and every accumulator sums half the K range.
// Same GemmSpec / grid conventions as gemm.cuh (strides and shapes in device memory,
// capacity-sized grid, surplus CTAs exit).
//
// CTA: 128 x 128 output tile, one tcgen05.mma.cta_group::1 M=128 N=128 K=8 per (k-step,
// term); K chunks of 32 staged by all 256 threads into SWIZZLE_NONE K-major core-matrix
// layouts (8 rows x 16 B cores; LBO = 128 B between K-adjacent cores, SBO = 1024 B between
// 8-row groups), double-buffered; one thread issues the MMAs and commits them to the
// buffer's mbarrier, so staging of chunk c+1 overlaps the MMAs of chunk c.  Epilogue: every
// warp reads its TMEM lane quadrant of the four accumulators (tcgen05.ld 32x32b), sums them
// in fp64 and writes fp64 C.
#pragma once
#include "gemm.cuh"

namespace qtt {

namespace tf32g {
constexpr int TM = 128, TN = 128, KC = 32;
constexpr int OPB = TM * KC * 4;                 // bytes of one operand tile (hi or lo) = 16 KB
constexpr int BUFB = 4 * OPB;                    // A_hi, A_lo, B_hi, B_lo = 64 KB
constexpr size_t SMEM_BYTES = 2 * BUFB + 1024;   // two buffers + barriers / TMEM address
}  // namespace tf32g

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// SWIZZLE_NONE K-major operand descriptor (sm_100 UMMA smem descriptor, version 1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                        // version (sm_100)
  return d;                                       // base offset 0, lbo mode 0, SWIZZLE_NONE
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = 128.
__host__ __device__ constexpr uint32_t tf32_idesc() {
  return (1u << 4)                 // c_format F32
       | (2u << 7)                 // a_format TF32
       | (2u << 10)                // b_format TF32
       | ((uint32_t)(tf32g::TN >> 3) << 17)
       | ((uint32_t)(tf32g::TM >> 4) << 24);
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}

// byte offset of element (row, k) of a 128 x 32 K-major core-matrix tile
__device__ __forceinline__ uint32_t core_off(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

template <bool A_KCONTIG>
__global__ void __launch_bounds__(256, 1) k_gemm_tf32(const GemmSpec *spec, int tiles_n, int nz2_cap) {
  using namespace tf32g;
  extern __shared__ __align__(1024) unsigned char tsm[];
  const GemmSpec g = *spec;
  const int z1 = blockIdx.z / nz2_cap, z2 = blockIdx.z % nz2_cap;
  if (z1 >= g.nz1 || z2 >= g.nz2) return;
  const int m0 = (blockIdx.x / tiles_n) * TM, n0 = (blockIdx.x % tiles_n) * TN;
  if (m0 >= g.M || n0 >= g.N) return;
  const double *A = g.A + z1 * g.sa1 + z2 * g.sa2;
  const double *B = g.B + z1 * g.sb1 + z2 * g.sb2;
  double *C = g.C + z1 * g.sc1 + z2 * g.sc2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char *buf0 = tsm;
  uint64_t *bars = reinterpret_cast<uint64_t *>(tsm + 2 * BUFB);   // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tsm + 2 * BUFB + 64);

  if (warp == 0) {   // 4 accumulators x TN columns = all 512 TMEM columns (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(4 * TN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  const int nk = (g.K + KC - 1) / KC;
  constexpr uint32_t idesc = tf32_idesc();
  for (int kc = 0; kc < nk; ++kc) {
    const int b = kc & 1;
    unsigned char *base = buf0 + b * BUFB;
    const int k0 = kc * KC;
    // global -> registers (fp64), before waiting for the buffer to drain
    double av[16], bv[16];
    if (A_KCONTIG) {                      // thread -> row tid/2, 16 consecutive k
      const int m = tid >> 1, kh = (tid & 1) * 16, gm = m0 + m;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int gk = k0 + kh + e;
        av[e] = (gm < g.M && gk < g.K) ? A[(long long)gm * g.sam + gk] : 0.0;
      }
    } else {                              // thread -> k = tid/8, 16 consecutive m
      const int k = tid >> 3, mh = (tid & 7) * 16, gk = k0 + k;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int gm = m0 + mh + e;
        av[e] = (gm < g.M && gk < g.K) ? A[(long long)gm * g.sam + (long long)gk * g.sak] : 0.0;
      }
    }
    {                                     // B: thread -> k = tid/8, 16 consecutive n
      const int k = tid >> 3, nh = (tid & 7) * 16, gk = k0 + k;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int gn = n0 + nh + e;
        bv[e] = (gn < g.N && gk < g.K) ? B[(long long)gk * g.sbk + (long long)gn * g.sbn] : 0.0;
      }
    }
    if (kc >= 2) mbar_wait(smem_u32(&bars[b]), ((kc >> 1) - 1) & 1);   // MMAs of chunk kc-2 done
    float *Ahi = reinterpret_cast<float *>(base), *Alo = reinterpret_cast<float *>(base + OPB);
    float *Bhi = reinterpret_cast<float *>(base + 2 * OPB), *Blo = reinterpret_cast<float *>(base + 3 * OPB);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      int row, k;
      if (A_KCONTIG) { row = tid >> 1; k = (tid & 1) * 16 + e; }
      else { row = (tid & 7) * 16 + e; k = tid >> 3; }
      const float x = (float)av[e], hi = tf32_rna(x), lo = tf32_rna(x - hi);
      const uint32_t o = core_off(row, k) >> 2;
      Ahi[o] = hi; Alo[o] = lo;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int nrow = (tid & 7) * 16 + e, k = tid >> 3;
      const float x = (float)bv[e], hi = tf32_rna(x), lo = tf32_rna(x - hi);
      const uint32_t o = core_off(nrow, k) >> 2;
      Bhi[o] = hi; Blo[o] = lo;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic stores -> tensor-core reads
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t sA = smem_u32(base), sAl = sA + OPB, sB = sA + 2 * OPB, sBl = sA + 3 * OPB;
#pragma unroll
      for (int s = 0; s < KC / 8; ++s) {
        const uint32_t off = s * 256;                 // two K-adjacent core matrices per MMA
        const uint64_t dAh = umma_desc(sA + off, 128, 1024), dAl = umma_desc(sAl + off, 128, 1024);
        const uint64_t dBh = umma_desc(sB + off, 128, 1024), dBl = umma_desc(sBl + off, 128, 1024);
        const uint64_t da[3] = {dAh, dAh, dAl}, db[3] = {dBh, dBl, dBh};
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          // accumulator: (hi*hi | corrections) x (chunk parity); first use of each overwrites
          const uint32_t slot = (t == 0 ? 0u : 1u) + 2u * (uint32_t)(kc & 1);
          const uint32_t acc = (kc > 1 || s > 0 || t == 2) ? 1u : 0u;
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + slot * TN),
              "l"(da[t]), "l"(db[t]), "r"(idesc), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(&bars[b]))
                   : "memory");
    }
  }
  // all MMAs done: the last commit covers every earlier tcgen05 op of the issuing thread
  if (nk > 0) mbar_wait(smem_u32(&bars[(nk - 1) & 1]), ((nk - 1) >> 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: warp w reads TMEM lanes 32*(w%4).. (rows), columns 64*(w/4) .. +63
  {
    const int q = warp & 3, half = warp >> 2;
    const int row = q * 32 + lane, gm = m0 + row;
#pragma unroll 1
    for (int cb = 0; cb < 64; cb += 16) {
      double sum[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) sum[e] = 0.0;
#pragma unroll
      for (int slot = 0; slot < 4; ++slot) {
        if (slot >= 2 && nk < 2) break;               // odd-chunk accumulators never written
        uint32_t r[16];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(slot * TN + half * 64 + cb);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int e = 0; e < 16; ++e) sum[e] += (double)__uint_as_float(r[e]);
      }
      if (gm < g.M) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int gn = n0 + half * 64 + cb + e;
          if (gn < g.N) C[(long long)gm * g.scm + (long long)gn * g.scn] = sum[e];
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(4 * TN));
}

}  // namespace qtt
