"""Factor time (median of reps) per push mode and zone budget (tuning build).
usage: push_sweep.py cfg reps modes(comma) zoneGB(comma, 0 = default)"""
import os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1908_10169_b200.build import build
os.environ["BILU_LIB"] = build(tuning=True)
from inputs.configs import make_config
from paper_1908_10169_b200 import BILU
name, reps = sys.argv[1], int(sys.argv[2])
modes = sys.argv[3].split(","); zbs = [int(float(z) * (1 << 30)) for z in sys.argv[4].split(",")]
P = make_config(name)
for zb in zbs:
    for mode in modes:
        os.environ["BILU_PUSH_MODE"] = mode
        g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm, zone_bytes=zb)
        g.factor(P.tau)
        ts = [g.factor(P.tau)["t_factor_ms"] for _ in range(reps)]
        st = g.factor(P.tau)
        print(name, "mode", mode, "zone GB %.0f" % (zb / 2**30), "median %.2f min %.2f max %.2f" % (np.median(ts), min(ts), max(ts)),
              "zone_blocks", st["zone_blocks"], flush=True)
        g.close()
