"""The library's CTA-level FP64 tensor-core GEMM (DMMA m8n8k4, csrc/dgemm_cta.cuh)
against a plain fp64 reference (torch CPU matmul), through the C-ABI diagnostic
entry bilu_diag_dgemm: ragged shapes, both operand layouts, alpha/beta."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1908_10169_b200.build import build
    build()


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (8, 8, 4), (64, 64, 16), (65, 63, 17), (200, 37, 128),
                                   (37, 130, 8), (5, 3, 129), (128, 128, 128), (0, 5, 5)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
@pytest.mark.parametrize("ts", [False, True])
def test_dgemm_matches_fp64_reference(M, N, K, ta, tb, ts):
    import torch
    from paper_1908_10169_b200.bilu import diag_dgemm
    g = torch.Generator().manual_seed(M * 1000 + N * 10 + K)
    bt = 3
    A = torch.randn(bt, K, M, generator=g, dtype=torch.float64).transpose(1, 2) if ta else \
        torch.randn(bt, M, K, generator=g, dtype=torch.float64)
    B = torch.randn(bt, N, K, generator=g, dtype=torch.float64).transpose(1, 2) if tb else \
        torch.randn(bt, K, N, generator=g, dtype=torch.float64)
    C0 = torch.randn(bt, M, N, generator=g, dtype=torch.float64)
    ref = -1.0 * (A @ B) + 0.5 * C0
    Ad, Bd, Cd = A.cuda(), B.cuda(), C0.clone().cuda()
    if ts and (N > 128 or K > 128):
        return
    diag_dgemm(Ad, Bd, Cd, alpha=-1.0, beta=0.5, tall_skinny=ts)
    torch.cuda.synchronize()
    out = Cd.cpu()
    if ref.numel() == 0:
        return
    tol = 1e-13 * max(1, K) * (ref.abs().max().item() + 1)
    assert (out - ref).abs().max().item() <= tol
