"""Run one factorization of a config (used under ncu)."""
import sys
sys.path.insert(0, "/root/repo")
from inputs.configs import make_config
from paper_1908_10169_b200 import BILU
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
kw = {}
if name == "c2s":
    P = make_config("c2", N=32, leaf=256)
else:
    P = make_config(name)
g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
for _ in range(reps):
    st = g.factor(P.tau)
print(name, "ms", st["t_factor_ms"], "flops", st["flops"], "launches", g.kernel_launches(), "retries(last)", st["n_retries"])
