// gemm_test.cu -- test entry for the GEMM kernels of the large-member path (gemm.cuh FP64
// DMMA, gemm_tf32.cuh 3xTF32 tcgen05), so tests can compare them with torch.matmul on their
// own.  Diagnostics library (libqttprobe.so); the product calls the kernels inside libqtt.
#include "../gemm.cuh"
#include "../gemm_tf32.cuh"

using namespace qtt;

// C (M x N, row-major) = A * B.  A: M x K row-major (a_kcontig) or K x M row-major (A^T
// given, i.e. M-contiguous); B: K x N row-major.  kind 0 = DMMA fp64, 1 = 3xTF32 tcgen05,
// 2 = DMMA fp64 with the TMA bulk feed of aligned interior tiles (gemm.cuh, TMA = true).
extern "C" int qtt_test_gemm(int kind, int M, int N, int K, const double *A, const double *B, double *C,
                             int a_kcontig, void *stream) {
  cudaStream_t s = (cudaStream_t)stream;
  GemmSpec h{};
  h.M = M; h.N = N; h.K = K; h.nz1 = 1; h.nz2 = 1;
  h.A = A; h.B = B; h.C = C;
  if (a_kcontig) { h.sam = K; h.sak = 1; } else { h.sam = 1; h.sak = M; }
  h.sbk = N; h.sbn = 1; h.scm = N; h.scn = 1;
  GemmSpec *d = nullptr;
  if (cudaMalloc(&d, sizeof(GemmSpec)) != cudaSuccess) return 1;
  cudaMemcpyAsync(d, &h, sizeof(h), cudaMemcpyHostToDevice, s);
  const int TMk = kind == 1 ? tf32g::TM : dgemm::TM, TNk = kind == 1 ? tf32g::TN : dgemm::TN;
  const int tm = (M + TMk - 1) / TMk, tn = (N + TNk - 1) / TNk;
  dim3 grid(tm * tn, 1, 1);
  if (kind == 0) {
    cudaFuncSetAttribute(k_gemm_dmma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dgemm::SMEM_BYTES);
    cudaFuncSetAttribute(k_gemm_dmma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dgemm::SMEM_BYTES);
    if (a_kcontig) k_gemm_dmma<true><<<grid, 256, dgemm::SMEM_BYTES, s>>>(d, tn, 1);
    else k_gemm_dmma<false><<<grid, 256, dgemm::SMEM_BYTES, s>>>(d, tn, 1);
  } else if (kind == 2) {
    cudaFuncSetAttribute(k_gemm_dmma<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dgemm::SMEM_BYTES);
    cudaFuncSetAttribute(k_gemm_dmma<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dgemm::SMEM_BYTES);
    if (a_kcontig) k_gemm_dmma<true, false, true><<<grid, 256, dgemm::SMEM_BYTES, s>>>(d, tn, 1);
    else k_gemm_dmma<false, false, true><<<grid, 256, dgemm::SMEM_BYTES, s>>>(d, tn, 1);
  } else {
    cudaFuncSetAttribute(k_gemm_tf32<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tf32g::SMEM_BYTES);
    cudaFuncSetAttribute(k_gemm_tf32<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tf32g::SMEM_BYTES);
    if (a_kcontig) k_gemm_tf32<true><<<grid, 256, tf32g::SMEM_BYTES, s>>>(d, tn, 1);
    else k_gemm_tf32<false><<<grid, 256, tf32g::SMEM_BYTES, s>>>(d, tn, 1);
  }
  int err = (int)cudaGetLastError();
  cudaStreamSynchronize(s);
  if (!err) err = (int)cudaGetLastError();
  cudaFree(d);
  return err;
}
