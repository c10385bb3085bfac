"""Full-size run of one BASELINE config: generation, analyze, factorization (timed),
statistics.  usage: python tools/run_full.py c3|c4|c5 [reps] [key=value ...]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from inputs.configs import make_config
from paper_1908_10169_b200 import BILU

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
kw = dict(a.split("=") for a in sys.argv[3:])
kw = {k: int(v) for k, v in kw.items()}
t = time.time(); P = make_config(name, **kw); tg = time.time() - t
t = time.time()
g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
ta = time.time() - t
out = {"config": name, "n": P.n, "nnz": P.nnz, "blocks": int(len(P.block_sizes)), "gen_s": tg, "analyze_s": ta}
for r in range(reps):
    st = g.factor(P.tau)
    out["factor_ms_%d" % r] = st["t_factor_ms"]
out.update({k: st[k] for k in ("t_merge_ms", "flops", "nnz_L", "nnz_U", "nnz_D", "n_blocks_final", "n_merges",
                              "n_retries", "n_near")})
kern = st["t_factor_ms"] - st["t_merge_ms"]
out["gflops_total"] = st["flops"] / (st["t_factor_ms"] * 1e-3) / 1e9
out["factor_kernel_ms"] = kern
print(json.dumps(out), flush=True)
