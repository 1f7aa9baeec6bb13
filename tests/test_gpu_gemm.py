"""GPU numerics of the large-member GEMM kernels against torch.matmul (fp64):
FP64 DMMA (gemm.cuh) to fp64 rounding, 3xTF32 tcgen05 (gemm_tf32.cuh) to fp32 accuracy.
Shapes span several tiles with ragged tails and both A layouts, and both operand feeds of the
DMMA kernel (kind 0: cp.async, the product's; kind 2: TMA bulk copies for interior aligned
tiles, cp.async for the others)."""
import ctypes
import os

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def probe():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return ctypes.CDLL(os.path.join(ROOT, "paper_2602_20226_b200", "lib", "libqttprobe.so"))


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("M,N,K,akc", [(128, 128, 32, 1), (300, 200, 77, 1), (257, 129, 256, 0),
                                       (64, 520, 512, 0), (1000, 64, 40, 1),
                                       # interior 16-byte aligned tiles: the DMMA kernel's TMA bulk feed
                                       # (both operands; A only on the ragged-N column of tiles; B only)
                                       (256, 384, 64, 0), (256, 256, 48, 1), (384, 200, 128, 1), (130, 256, 32, 0)])
def test_gemm_kernels(probe, kind, M, N, K, akc):
    import torch
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(K, N, dtype=torch.float64, device="cuda", generator=g)
    C = torch.full((M, N), float("nan"), dtype=torch.float64, device="cuda")
    Ain = A.contiguous() if akc else A.t().contiguous()          # M-contiguous storage of A
    st = torch.cuda.current_stream()
    rc = probe.qtt_test_gemm(kind, M, N, K, ctypes.c_void_p(Ain.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                             ctypes.c_void_p(C.data_ptr()), akc, ctypes.c_void_p(st.cuda_stream))
    assert rc == 0
    ref = A @ B
    scale = (A.abs() @ B.abs()).max().item()
    err = (C - ref).abs().max().item() / scale
    tol = 1e-14 * K if kind != 1 else 5e-7           # fp64 rounding / 3xTF32 (measured <= 1.7e-7)
    print(f"kind {kind} M{M} N{N} K{K} err {err:.3e}")
    assert err <= tol, (kind, err)
