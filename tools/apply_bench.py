"""Time bilu_apply (the preconditioner solve) on a config: CUDA events,
mean of 20 applies after 3 warm-up.  usage: python tools/apply_bench.py c2 [key=value ...]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from inputs.configs import make_config
from paper_1908_10169_b200 import BILU
name = sys.argv[1]
kw = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
P = make_config(name, **kw)
g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
st = g.factor(P.tau)
x = torch.ones(P.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    y = g.apply_tensor(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    y = g.apply_tensor(x)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
nb = 8.0 * (st["nnz_L"] + st["nnz_U"] + st["nnz_D"])
print(json.dumps({"config": name, "apply_ms": ms, "factor_bytes": nb, "GB/s": nb / (ms * 1e-3) / 1e9,
                  "blocks_final": st["n_blocks_final"]}))
