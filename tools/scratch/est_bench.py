"""ILU(1,tau) initial blocking on the device: estimate time vs the oracle's, and the factorization
from the estimated partition vs the configs' stand-in blocking.  python tools/est_bench.py c2 c3 c5"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: timed beside the device path)
from inputs.configs import make_config  # noqa: E402
from paper_1908_10169_b200 import BILU, cosine_blocks, ilu1_blocks  # noqa: E402

for name in sys.argv[1:] or ["c2"]:
    P = make_config(name)
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm) if P.perm is not None else (
        P.indptr, P.indices, P.data)
    ts = []
    for _ in range(4):
        t = time.perf_counter()
        bs, nl = ilu1_blocks(ip, ix, dv, P.tau, 8)
        ts.append(time.perf_counter() - t)
    t = time.perf_counter()
    ob = oracle.ilu1_blocks(ip, ix, dv, P.tau, 8)
    to = time.perf_counter() - t
    assert np.array_equal(bs, ob)
    print("%s n=%d nnz=%d estimate: device API %.1f ms (min of 3 after warm-up, %d launches), oracle %.0f ms; "
          "%d blocks, sizes %s" % (name, P.n, len(ix), 1e3 * min(ts[1:]), nl, 1e3 * to, len(bs),
                                   np.bincount(bs).tolist()), flush=True)
    ts = []
    for _ in range(4):
        t = time.perf_counter()
        cq, cs, cl = cosine_blocks(P.indptr, P.indices, 0.8, 128)
        ts.append(time.perf_counter() - t)
    t = time.perf_counter()
    oq, os_ = oracle.cosine_blocks(P.indptr, P.indices, 0.8, 128)
    to = time.perf_counter() - t
    assert np.array_equal(cq, oq) and np.array_equal(cs, os_)
    print("%s cosine blocking: device API %.1f ms (%d launches), oracle %.0f ms; %d groups, sizes %s" % (
        name, 1e3 * min(ts[1:]), cl, 1e3 * to, len(cs), np.bincount(cs).tolist()[:10]), flush=True)
    if os.environ.get("EST_NO_FACTOR"):
        continue
    for label, blocks in (("stand-in", P.block_sizes), ("ilu1", bs)):
        g = BILU(P.indptr, P.indices, P.data, blocks, perm=P.perm)
        for _ in range(2):
            st = g.factor(P.tau)
        b = torch.ones(P.n, dtype=torch.float64, device="cuda")
        x, sst = g.gmres(b, restart=30, tol=1e-8, max_restarts=20)
        print("  %-8s init %7d final %7d merges %7d factor %.1f ms (merge %.1f) %.1f GFLOP  gmres %d it" % (
            label, st["n_blocks_init"], st["n_blocks_final"], st["n_merges"], st["t_factor_ms"], st["t_merge_ms"],
            st["flops"] / 1e9, sst["iterations"]), flush=True)
        del g
