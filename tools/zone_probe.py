"""Factor time vs dense-trailing-zone budget: python tools/zone_probe.py c5 [reps] [GiB,GiB,...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs.configs import make_config
from paper_1908_10169_b200 import BILU
name = sys.argv[1]; reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
P = make_config(name)
zbs = [int(float(x) * (1 << 30)) for x in sys.argv[3].split(',')] if len(sys.argv) > 3 else [-1, 64 << 20, 256 << 20, 1 << 30, 4 << 30, 0]
for zb in zbs:
    try:
        g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm, zone_bytes=zb)
    except Exception as e:   # e.g. the budget does not fit the free HBM
        print("%s zone_bytes=%d: %s" % (name, zb, e), flush=True)
        continue
    ts = []
    for _ in range(reps):
        st = g.factor(P.tau)
        ts.append(st["t_factor_ms"])
    print("%s zone_bytes=%d: zone %d blocks / %d unknowns, ms %s, merge %.2f, flops %.6g" % (
        name, zb, st["zone_blocks"], st["zone_unknowns"], " ".join("%.2f" % t for t in ts), st["t_merge_ms"], st["flops"]),
        flush=True)
    g.close()
