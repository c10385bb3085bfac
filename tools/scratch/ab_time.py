"""A/B factor time of two library builds on one config (median of reps, interleaved).
usage: ab_time.py cfg reps libA libB"""
import os, sys, subprocess, json
cfg, reps, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
code = r'''
import os, sys, json
sys.path.insert(0, "/root/repo")
from inputs.configs import make_config
from paper_1908_10169_b200 import BILU
P = make_config(sys.argv[1])
g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
g.factor(P.tau)
print(json.dumps([g.factor(P.tau)["t_factor_ms"] for _ in range(int(sys.argv[2]))]))
'''
import numpy as np
res = {l: [] for l in libs}
for rnd in range(2):
    for l in libs:
        out = subprocess.run([sys.executable, "-c", code, cfg, str(reps)], env=dict(os.environ, BILU_LIB=l),
                             capture_output=True, text=True).stdout.strip().splitlines()[-1]
        res[l] += json.loads(out)
for l in libs:
    t = np.array(res[l])
    print(cfg, os.path.basename(l), "median %.2f mean %.2f min %.2f max %.2f n %d" % (np.median(t), t.mean(), t.min(), t.max(), len(t)))
