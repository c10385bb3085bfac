"""Analyze a factor_kernel per-block profile (tools/block_profile.py output) by ND level of c2:
top separator (last 4096 unknowns), level-2 separators, the rest."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
fn = sys.argv[1]
a = np.load(fn)
cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
from inputs.configs import make_config
P = make_config(cfg)
bs = np.concatenate([[0], np.cumsum(P.block_sizes)])
n = bs[-1]
t0 = a[:, 0].min(); st = (a[:, 0] - t0) / 1e3; en = (a[:, 10] - t0) / 1e3
ph = a[:, 2:10] / 1965.
names = ["contrib", "Lprep", "Uprep", "upd", "pivot", "drop", "reg", "release"]
sub = a[:, 16:32] / 1965.
Z = np.searchsorted(bs, n - 4096); Z2 = np.searchsorted(bs, n - 8192)
for nm, sel in (("top sep", np.arange(Z, len(bs) - 1)), ("lvl2", np.arange(Z2, Z)), ("rest", np.arange(0, Z2))):
    print("%s: %d blocks, span %.0f-%.0f us, dur mean %.1f" % (nm, len(sel), st[sel].min(), en[sel].max(), (en - st)[sel].mean()))
    print("   phases", {k: round(float(ph[sel, i].mean()), 1) for i, k in enumerate(names)})
    print("   sub (16+i)", {i: round(float(sub[sel, i].mean()), 1) for i in range(16) if sub[sel, i].mean() > 0.05})
    print("   nR %.1f nC %.1f" % (a[sel, 13].mean(), a[sel, 14].mean()))
print("total span %.2f ms" % (en.max() / 1e3))
