"""Critical path of a factor_kernel per-block profile: walk back from the last block through the
latest-finishing contributor (DAG from the oracle's unaggregated structure, cached in /tmp)."""
import sys, os
import numpy as np
sys.path.insert(0, "/root/repo")
fn = sys.argv[1]; cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
cache = "/tmp/%s_struct.npz" % cfg
if not os.path.exists(cache):
    import oracle
    from inputs.configs import make_config
    P = make_config(cfg)
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    f = oracle.factor(ip, ix, dv, P.block_sizes, P.tau, aggregate=False)
    np.savez(cache, bstart=f.bstart, Lp=f.Lp, Li=f.Li, Up=f.Up, Ui=f.Ui)
d = np.load(cache); bs = d["bstart"]; Lp = d["Lp"]; Li = d["Li"]; Up = d["Up"]; Ui = d["Ui"]
nb = len(bs) - 1; n = bs[-1]
blk = np.repeat(np.arange(nb), np.diff(bs))
pred = [set() for _ in range(nb)]
for J in range(nb):
    for T in np.unique(blk[Li[Lp[J]:Lp[J + 1]]]): pred[T].add(J)
    for T in np.unique(blk[Ui[Up[J]:Up[J + 1]]]): pred[T].add(J)
a = np.load(fn)
t0 = a[:, 0].min(); st = (a[:, 0] - t0) / 1e3; en = (a[:, 10] - t0) / 1e3
K = int(np.argmax(en)); path = []
while True:
    path.append(K)
    if not pred[K]: break
    K = max(pred[K], key=lambda J: en[J])
path = path[::-1]
path = np.array(path)
durs = en[path] - st[path]
gaps = np.array([st[path[i]] - en[path[i - 1]] for i in range(1, len(path))])
print("critical path: %d blocks, ends at %.2f ms; block time %.2f ms (mean %.1f us), gaps %.2f ms (mean %.1f us)" % (
    len(path), en[path[-1]] / 1e3, durs.sum() / 1e3, durs.mean(), gaps.sum() / 1e3, gaps.mean()))
Z = np.searchsorted(bs, n - 4096); Z2 = np.searchsorted(bs, n - 8192)
for nm, lo, hi in (("top sep", Z, nb), ("lvl2", Z2, Z), ("rest", 0, Z2)):
    m = (path >= lo) & (path < hi)
    print("  %-8s %4d blocks on the path, block time %.2f ms, mean %.1f us" % (nm, m.sum(), durs[m].sum() / 1e3, durs[m].mean() if m.any() else 0))

# the scheduler's DAG: static block adjacency of sym(Ã) + chain edges of every N(J)
from inputs.configs import make_config
import oracle, scipy.sparse as sp
P = make_config(cfg)
ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
A = sp.csr_matrix((dv, ix, ip), shape=(n, n)).tocoo()
bi, bj = blk[A.row], blk[A.col]
m = bi != bj
lo_, hi_ = np.minimum(bi[m], bj[m]), np.maximum(bi[m], bj[m])
spred = [set() for _ in range(nb)]
for x, y in set(zip(lo_.tolist(), hi_.tolist())): spred[y].add(x)
for J in range(nb):
    NJ = np.unique(np.concatenate([blk[Li[Lp[J]:Lp[J + 1]]], blk[Ui[Up[J]:Up[J + 1]]]]))
    for x, y in zip(NJ[:-1], NJ[1:]): spred[y].add(int(x))
    if len(NJ): spred[NJ[0]].add(J)
K = int(np.argmax(en)); path = []
while True:
    path.append(K)
    if not spred[K]: break
    K = max(spred[K], key=lambda J: en[J])
path = np.array(path[::-1])
durs = en[path] - st[path]
gaps = np.array([st[path[i]] - en[path[i - 1]] for i in range(1, len(path))])
print("scheduler critical path: %d blocks, block time %.2f ms (mean %.1f us), gaps %.2f ms (mean %.1f us, median %.1f)" % (
    len(path), durs.sum() / 1e3, durs.mean(), gaps.sum() / 1e3, gaps.mean(), np.median(gaps)))
for nm, lo, hi in (("top sep", Z, nb), ("lvl2", Z2, Z), ("rest", 0, Z2)):
    mm = (path >= lo) & (path < hi)
    print("  %-8s %4d blocks on the path, block time %.2f ms, mean %.1f us" % (nm, mm.sum(), durs[mm].sum() / 1e3, durs[mm].mean() if mm.any() else 0))
zb = int(sys.argv[3]) if len(sys.argv) > 3 else 0
if zb:
    Zz = nb - zb
    mm = path >= Zz
    print("  zone (last %d blocks): %d on the path, mean %.1f us; non-zone %d, mean %.1f us" % (zb, mm.sum(), durs[mm].mean() if mm.any() else 0, (~mm).sum(), durs[~mm].mean()))
    # where are the non-zone path blocks: histogram of their position
    pos = path[~mm]
    print("  non-zone path blocks: first %d last %d; unknown ranges" % (pos.min(), pos.max()), np.percentile(bs[pos], [0, 25, 50, 75, 100]).astype(int), "n", n)
    ph = a[:, 2:10] / 1965.
    names = ["contrib", "Lprep", "Uprep", "upd", "pivot", "drop", "reg", "release"]
    print("  non-zone path phases", {k: round(float(ph[pos, i].mean()), 1) for i, k in enumerate(names)})
    print("  zone path phases", {k: round(float(ph[path[mm], i].mean()), 1) for i, k in enumerate(names)})

def zone_of(nzb_target):
    """zone = the nzb_target blocks with the largest etree subtrees (bilu_host.cpp zone selection)"""
    par = np.full(nb, -1); anc = np.full(nb, -1)
    lower = [[] for _ in range(nb)]
    for y in range(nb):
        for x in spred_static[y]: lower[y].append(x)
    for K in range(nb):
        for r in lower[K]:
            while anc[r] != -1 and anc[r] != K:
                nx = anc[r]; anc[r] = K; r = nx
            if anc[r] == -1: anc[r] = K; par[r] = K
    sub = np.diff(bs).astype(np.int64)
    for K in range(nb):
        if par[K] >= 0: sub[par[K]] += sub[K]
    order = sorted(range(nb), key=lambda x: (-sub[x], -x))
    z = np.zeros(nb, bool); z[order[:nzb_target]] = True
    return z
if len(sys.argv) > 4:
    spred_static = [set() for _ in range(nb)]
    for x, y in set(zip(lo_.tolist(), hi_.tolist())): spred_static[y].add(x)
    z = zone_of(int(sys.argv[4]))
    mm = z[path]
    print("  etree zone (%d blocks): %d on the path, block time %.2f ms (mean %.1f us); non-zone %d, %.2f ms (mean %.1f us)" % (
        z.sum(), mm.sum(), durs[mm].sum() / 1e3, durs[mm].mean(), (~mm).sum(), durs[~mm].sum() / 1e3, durs[~mm].mean()))
    # gaps before zone / non-zone blocks
    g2 = np.concatenate([[0], gaps])
    print("  gaps before zone blocks %.2f ms, before non-zone %.2f ms" % (g2[mm].sum() / 1e3, g2[~mm].sum() / 1e3))
    ph = a[:, 2:10] / 1965.
    names = ["contrib", "Lprep", "Uprep", "upd", "pivot", "drop", "reg", "release"]
    print("  zone path phases", {k: round(float(ph[path[mm], i].mean()), 1) for i, k in enumerate(names)})
    print("  non-zone path phases", {k: round(float(ph[path[~mm], i].mean()), 1) for i, k in enumerate(names)})
if len(sys.argv) > 4:
    g2 = np.concatenate([[0], gaps])
    big = np.argsort(-g2)[:15]
    print("  largest gaps on the path (start ms, gap us, zone?):", [(round(st[path[i]] / 1e3, 2), round(g2[i], 1), bool(z[path[i]])) for i in sorted(big)])
    tt = st[path] / 1e3
    for lo, hi in ((0, 10), (10, 20), (20, 30), (30, 60)):
        m2 = (tt >= lo) & (tt < hi)
        print("  path blocks starting in [%d, %d) ms: %d, gaps %.2f ms, block time %.2f ms" % (lo, hi, m2.sum(), g2[m2].sum() / 1e3, durs[m2].sum() / 1e3))
    # concurrency over time
    ts = np.linspace(0, en.max(), 12)
    print("  active blocks:", [int(((st <= t) & (en > t)).sum()) for t in ts])
