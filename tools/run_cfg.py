"""Factor one config (reps times) with keyword overrides: python tools/run_cfg.py c4 2 nblocks=2000"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs.configs import make_config
from paper_1908_10169_b200 import BILU
name = sys.argv[1]; reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
kw = {k: int(v) for k, v in (a.split("=") for a in sys.argv[3:])}
P = make_config(name, **kw)
g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
for _ in range(reps):
    st = g.factor(P.tau)
print(name, kw, "ms", st["t_factor_ms"], "merge", st["t_merge_ms"], "flops", st["flops"])
