"""Quick GPU-vs-oracle parity sweep (development tool; the real gates are tests/)."""
import sys, time, traceback
import numpy as np
sys.path.insert(0, "/root/repo")
import oracle
from inputs.configs import config1, config2, random_dd, dense_to_csr
from paper_1908_10169_b200 import BILU
from tests.parity import compare_factors, oracle_replay, overrides_from_near


def run(name, ip, ix, dv, bs, tau, agg, perm=None):
    t = time.time()
    g = BILU(ip, ix, dv, bs, perm=perm, aggregate=int(agg))
    st = g.factor(tau)
    st = g.factor(tau)
    gf = g.export()
    if perm is not None:
        pip, pix, pdv = oracle.permute_csr(ip, ix, dv, perm)
    else:
        pip, pix, pdv = ip, ix, dv
    ov = overrides_from_near(gf.near)
    of = oracle_replay(pip, pix, pdv, bs, tau, aggregate=agg, overrides=ov)
    r = compare_factors(gf, of)
    print("%-28s tau=%-6g agg=%d  blocks %5d->%5d  gpu %.3f ms  oracle %.3f s  flops g/o %.4g/%.4g  near %d  max_rel %.2e  %s" % (
        name, tau, agg, len(bs), gf.nblk, st["t_factor_ms"], of.t_factor_s, st["flops"], of.flops,
        len(gf.near), r["max_rel"], "OK" if not r["problems"] else r["problems"][:3]), flush=True)
    # apply
    import torch
    x = torch.ones(len(ip) - 1, dtype=torch.float64, device="cuda")
    y = g.apply_tensor(x).cpu().numpy()
    xo = np.ones(len(ip) - 1)
    if perm is not None:
        yo_p = oracle.apply(of, xo[perm])
        yo = np.empty_like(yo_p); yo[perm] = yo_p
    else:
        yo = oracle.apply(of, xo)
    print("    apply max rel diff %.2e" % (np.abs(y - yo).max() / np.abs(yo).max()), flush=True)
    g.close()


cases = sys.argv[1:] or ["small", "c1", "c2"]
try:
    if "small" in cases:
        for seed, n, bsz in [(0, 12, [3, 4, 5]), (1, 40, [3, 5, 2, 4, 6, 1, 3, 8, 4, 4]), (2, 200, [8] * 25)]:
            A = random_dd(n, 0.15, seed)
            ip, ix, dv = dense_to_csr(A)
            for tau in [0.0, 1e-2, 0.1]:
                for agg in [False, True]:
                    run("rand n=%d seed=%d" % (n, seed), ip, ix, dv, np.array(bsz), tau, agg)
    if "c1" in cases:
        P = config1()
        for agg in [False, True]:
            run("c1", P.indptr, P.indices, P.data, P.block_sizes, P.tau, agg, P.perm)
    if "c2" in cases:
        P = config2()
        for agg in [False, True]:
            run("c2", P.indptr, P.indices, P.data, P.block_sizes, P.tau, agg, P.perm)
except Exception:
    traceback.print_exc()
    sys.exit(1)
