"""Factor a config from its ILU(1,tau) partition (many small blocks -> many merges).
python tools/merge_probe.py c2 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs.configs import make_config  # noqa: E402
from paper_1908_10169_b200 import BILU, ilu1_blocks  # noqa: E402

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
P = make_config(name)
bs, _ = ilu1_blocks(P.indptr, P.indices, P.data, P.tau, 8, perm=P.perm)
g = BILU(P.indptr, P.indices, P.data, bs, perm=P.perm)
for _ in range(reps):
    st = g.factor(P.tau)
print(name, "ilu1 blocks", len(bs), "ms", st["t_factor_ms"], "merge", st["t_merge_ms"], "merges", st["n_merges"])
