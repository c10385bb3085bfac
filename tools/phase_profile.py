"""Per-phase cycle counters of factor_kernel (diagnostic build libbilu_prof.so)."""
import ctypes, os, sys
sys.path.insert(0, "/root/repo")
os.environ["BILU_LIB"] = "/root/repo/paper_1908_10169_b200/libbilu_prof.so"
import numpy as np
from inputs.configs import make_config
from paper_1908_10169_b200 import BILU
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
P = make_config(name)
g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm, aggregate=0)
g.factor(P.tau)
buf = (ctypes.c_ulonglong * 32)()
g.lib.bilu_prof_read(buf, 1)
st = g.factor(P.tau)
g.lib.bilu_prof_read(buf, 0)
names = ["pop-wait", "contributors", "L: hash/scatter/bucket", "L: updates", "U side (all)", "pivot inverse",
         "scale/drop/compact", "registration+chains", "release"]
nb = buf[31]
tot = sum(buf[i] for i in range(len(names)))
print("%s: blocks %d, factor %.2f ms, flops %.3g" % (name, nb, st["t_factor_ms"], st["flops"]))
for i, nm in enumerate(names):
    print("  %-22s %8.2f us/block  %5.1f%%" % (nm, buf[i] / nb / 1965.0, 100.0 * buf[i] / tot))
