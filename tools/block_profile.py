"""Per-block timeline of factor_kernel (diagnostic build): where does the critical path go?"""
import ctypes, os, sys, json
sys.path.insert(0, "/root/repo")
os.environ["BILU_LIB"] = "/root/repo/paper_1908_10169_b200/libbilu_prof.so"
import numpy as np, torch
from inputs.configs import make_config
from paper_1908_10169_b200 import BILU
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
P = make_config(name)
nct = int(sys.argv[2]) if len(sys.argv) > 2 else 0
zb = int(float(sys.argv[3]) * (1 << 30)) if len(sys.argv) > 3 else 0
g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm, aggregate=0, n_ctas=nct, zone_bytes=zb)
N = len(P.block_sizes)
buf = torch.zeros(N * 32, dtype=torch.int64, device="cuda")
g.lib.bilu_prof_set_blk(ctypes.c_void_p(buf.data_ptr()))
g.factor(P.tau)
buf.zero_()
torch.cuda.synchronize()
st = g.factor(P.tau)
a = buf.cpu().numpy().reshape(N, 32).astype(np.float64)
np.save("/root/repo/gpurun_out/blkprof_%s.npy" % name, a)
t0 = a[:, 0].min()
start = (a[:, 0] - t0) / 1e3; end = (a[:, 10] - t0) / 1e3
dur = end - start
print("n_ctas=%d" % nct); print("%s: factor %.2f ms, span of block times %.2f ms" % (name, st["t_factor_ms"], end.max() / 1e3))
print("block duration us: mean %.1f p50 %.1f p90 %.1f max %.1f" % (dur.mean(), np.median(dur), np.percentile(dur, 90), dur.max()))
ts = np.linspace(0, end.max(), 20)
conc = [int(((start <= t) & (end > t)).sum()) for t in ts]
print("active blocks over time:", conc)
names = ["contrib", "Lprep", "Uprep", "upd", "pivot", "drop", "reg", "release"]
ph = a[:, 2:10] / 1965.0
heavy = np.argsort(-dur)[:200]
print("heaviest 200 blocks: mean dur %.1f us; phase us:" % dur[heavy].mean(), {n: round(float(ph[heavy, i].mean()), 1) for i, n in enumerate(names)})
print("  sizes nLc %.1f nUc %.1f nR %.1f nC %.1f" % tuple(a[heavy, 11:15].mean(axis=0)))
light = np.argsort(dur)[:N // 2]
print("lightest half: mean dur %.1f us; phase us:" % dur[light].mean(), {n: round(float(ph[light, i].mean()), 1) for i, n in enumerate(names)})
print("  sizes nLc %.1f nUc %.1f nR %.1f nC %.1f" % tuple(a[light, 11:15].mean(axis=0)))
late = np.argsort(start)[-300:]
print("last 300 started blocks: mean dur %.1f us" % dur[late].mean())

sub = ["candidates", "W init+A", "updates"]
for side in (0, 1):
    print("side %d heavy sub-phases us:" % side, {n: round(float(a[heavy, 16 + 8 * side + i].mean() / 1965.0), 1) for i, n in enumerate(sub)})
# split heavy blocks: publish time (19), first part start (20), last part end (21), parts (22), part cycles (23)
sp = a[:, 22] > 0
if sp.any():
    pub = (a[sp, 19] - t0) / 1e3; f0 = (a[sp, 20] - t0) / 1e3; f1 = (a[sp, 21] - t0) / 1e3
    fin = end[sp]
    print("split blocks %d: owner %.1f us, publish->first part %.1f us, part span %.1f us, last part->finish end %.1f us, parts %.1f, us/part %.1f" % (
        sp.sum(), (pub - start[sp]).mean(), (f0 - pub).mean(), (f1 - f0).mean(), (fin - f1).mean(), a[sp, 22].mean(),
        (a[sp, 23] / a[sp, 22] / 1965.0).mean()))
