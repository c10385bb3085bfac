"""Throughput of the library's FP64 tensor-core GEMM routines on their own (one CTA per
product, batch = multiple of 148): the Schur-update shape (tall-skinny: M x K panel times a
K x N block, K, N = b_J, b <= 128) and square 64-tiled products.  CUDA events, best of 5."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1908_10169_b200.bilu import diag_dgemm

PEAK = 37.2
out = []
for (M, N, K, ts, batch) in [(2048, 64, 64, True, 148 * 4), (4096, 32, 32, True, 148 * 4), (2048, 48, 48, True, 148 * 4),
                             (1024, 128, 128, True, 148 * 2), (512, 512, 64, False, 148 * 2), (256, 256, 256, False, 148 * 2)]:
    A = torch.randn(batch, M, K, dtype=torch.float64, device="cuda")
    B = torch.randn(batch, K, N, dtype=torch.float64, device="cuda")
    C = torch.zeros(batch, M, N, dtype=torch.float64, device="cuda")
    diag_dgemm(A, B, C, tall_skinny=ts)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); diag_dgemm(A, B, C, tall_skinny=ts); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    ref = torch.bmm(A[:2], B[:2])
    err = (C[:2] - ref).abs().max().item() / ref.abs().max().item()
    tf = 2.0 * M * N * K * batch / (best * 1e-3) / 1e12
    r = {"kernel": "cta_tsgemm" if ts else "cta_dgemm", "M": M, "N": N, "K": K, "batch": batch, "ms": best,
         "TFLOP/s": round(tf, 2), "frac_fp64_peak": round(tf / PEAK, 3), "rel_err": err}
    out.append(r); print(json.dumps(r), flush=True)
# cuBLAS DGEMM on the same tall-skinny shape, for context
A = torch.randn(148 * 4, 2048, 64, dtype=torch.float64, device="cuda"); B = torch.randn(148 * 4, 64, 64, dtype=torch.float64, device="cuda")
torch.bmm(A, B); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); torch.bmm(A, B); e1.record(); torch.cuda.synchronize()
print(json.dumps({"kernel": "cuBLAS bmm (context)", "M": 2048, "N": 64, "K": 64, "batch": 592,
                  "TFLOP/s": round(2.0 * 2048 * 64 * 64 * 592 / (e0.elapsed_time(e1) * 1e-3) / 1e12, 2)}))
