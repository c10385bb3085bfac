"""Critical path of the two apply sweeps from per-block device timestamps (BILU_APPLY_PROF).
For each sweep: the last block to finish, walked back through the dependency released last
(the one that made it ready); the path time is split into queue wait (ready -> popped), work
(popped -> computed) and release.  usage: python tools/apply_profile.py c2"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_10169_b200.build import build  # noqa: E402
os.environ["BILU_LIB"] = build(tuning=True)   # BILU_APPLY_PROF is read by the tuning build only
import torch  # noqa: E402
from inputs.configs import make_config  # noqa: E402
from paper_1908_10169_b200 import BILU  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
P = make_config(name)
g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
g.factor(P.tau)
x = torch.ones(P.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    g.apply_tensor(x)
path = "/tmp/apply_prof"
os.environ["BILU_APPLY_PROF"] = path
g.apply_tensor(x)
torch.cuda.synchronize()
del os.environ["BILU_APPLY_PROF"]
f = g.export()
bs = np.asarray(f.bstart)
nF = len(bs) - 1
blk = np.searchsorted(bs, np.arange(bs[-1]), side="right") - 1
b = np.diff(bs)
mL, cU = np.diff(np.asarray(f.Lp)), np.diff(np.asarray(f.Up))
Li, Ui, Lp, Up = np.asarray(f.Li), np.asarray(f.Ui), np.asarray(f.Lp), np.asarray(f.Up)
preds = {"fwd": [[] for _ in range(nF)], "bwd": [[] for _ in range(nF)]}
for J in range(nF):
    for T in np.unique(blk[Li[Lp[J]:Lp[J + 1]]]):
        preds["fwd"][T].append(J)        # T waits for J's push
    for T in np.unique(blk[Ui[Up[J]:Up[J + 1]]]):
        preds["bwd"][J].append(T)        # J pulls from T
for sw in ("fwd", "bwd"):
    t = np.fromfile(path + "." + sw, dtype=np.uint64).reshape(nF, 3).astype(np.float64)
    t0 = t[t[:, 0] > 0, 0].min()
    t = (t - t0) / 1e3                    # us
    total = t[:, 2].max()
    k = int(np.argmax(t[:, 2]))
    chain, wait, work, rel = [], 0.0, 0.0, 0.0
    while True:
        chain.append(k)
        work += t[k, 1] - t[k, 0]
        rel += t[k, 2] - t[k, 1]
        pr = preds[sw][k]
        if not pr:
            wait += t[k, 0]
            break
        p = max(pr, key=lambda j: t[j, 2])
        wait += max(0.0, t[k, 0] - t[p, 2])
        k = p
    ch = np.array(chain)
    w = t[ch, 1] - t[ch, 0]
    print("%s %s: sweep %.0f us, critical path %d blocks: queue wait %.0f us, work %.0f us, release %.0f us" % (
        name, sw, total, len(ch), wait, work, rel))
    print("   per path block: work mean %.1f us (max %.1f), b mean %.1f, %s mean %.0f" % (
        w.mean(), w.max(), b[ch].mean(), "L rows" if sw == "fwd" else "U cols",
        (mL if sw == "fwd" else cU)[ch].mean()))
    top = np.argsort(-w)[:5]
    print("   heaviest on path:", [(int(ch[i]), int(b[ch[i]]), int((mL if sw == 'fwd' else cU)[ch[i]]), round(float(w[i]), 1)) for i in top])
