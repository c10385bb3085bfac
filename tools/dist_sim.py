"""Simulated multi-GPU run on one GPU: every rank's context runs its phases one after another
(phase A of all ranks, the interface exchange by device-to-device handover, phase B of all
ranks).  Checks the union of the ranks' factors against the oracle run with the same
aggregation segments, and projects the N-GPU time: a rank owns a whole GPU, so its phase
timings measured alone on this GPU are what it would see; the exchange is projected from
the packed bytes at NVLink 5 bandwidth (~900 GB/s per direction).
usage: python tools/dist_sim.py c2 8 [--no-oracle]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from inputs.configs import make_config
from paper_1908_10169_b200 import BILU
from paper_1908_10169_b200.dist import partition_owner

name, world = sys.argv[1], int(sys.argv[2])
check = "--no-oracle" not in sys.argv
P = make_config(name, top_levels=int(round(np.log2(world))))
owner = partition_owner(P.block_part, world)
ctxs = [BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm) for _ in range(world)]
for r, g in enumerate(ctxs):
    g.dist_setup(owner, r)


def run_once():
    ta = [g.factor_local(P.tau)["t_factor_ms"] for g in ctxs]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bufs = [g.interface_pack() for g in ctxs]
    for r, g in enumerate(ctxs):
        for q in range(world):
            if q != r:
                g.interface_unpack(bufs[q])
    torch.cuda.synchronize()
    t_ex_sim = (time.perf_counter() - t0) * 1e3
    stb = [g.factor_separators() for g in ctxs]
    tb = [s["t_factor_ms"] - ta[r] for r, s in enumerate(stb)]
    return ta, tb, [b.numel() for b in bufs], t_ex_sim, stb


run_once()
ta, tb, nbytes, t_ex_sim, stb = run_once()
single = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
single.factor(P.tau)
t1 = single.factor(P.tau)["t_factor_ms"]
recv = [sum(nbytes) - nbytes[r] for r in range(world)]
t_ex = max(recv) / 900e9 * 1e3
proj = max(ta) + t_ex + max(tb)
out = {"config": name, "world": world, "phaseA_ms_per_rank": [round(x, 2) for x in ta],
       "phaseB_ms": round(max(tb), 2), "exchange_bytes_per_rank": nbytes,
       "exchange_ms_projected_nvlink": round(t_ex, 4), "projected_ms": round(proj, 2),
       "single_gpu_ms": round(t1, 2), "projected_speedup": round(t1 / proj, 3)}
# distributed apply: each rank's begin / end timed alone (CUDA events), the two all-reduces
# projected (separator contributions, then y) at NVLink bandwidth + 15 us latency each
def ev_time(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    r = fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b), r


x = torch.ones(P.n, dtype=torch.float64, device="cuda")
for _ in range(2):
    tbeg, contribs = zip(*[ev_time(lambda g=g: g.apply_dist_begin(x)) for g in ctxs])
    total = sum(c.clone() for c in contribs)
    tend, ys = zip(*[ev_time(lambda r=r, g=g: g.apply_dist_end(total, r == 0)) for r, g in enumerate(ctxs)])
y_dist = sum(ys)
m = contribs[0].numel()
t_ar = 2 * 15e-3 + (m * 8 + P.n * 8) / 900e9 * 1e3
ya = torch.empty_like(x)
for _ in range(3):
    t_single_apply, _ = ev_time(lambda: single.apply(x.data_ptr(), ya.data_ptr()))
out.update({"apply_begin_ms_per_rank": [round(v, 3) for v in tbeg], "apply_end_ms_per_rank": [round(v, 3) for v in tend],
            "apply_separator_rows": m, "apply_allreduce_ms_projected": round(t_ar, 4),
            "apply_projected_ms": round(max(tbeg) + t_ar + max(tend), 3),
            "apply_single_gpu_ms": round(t_single_apply, 3)})
if check:
    import oracle
    from tests.parity import compare_present_blocks, oracle_replay
    exports = [g.export() for g in ctxs]
    near = {tuple(int(x) for x in row) for f in exports for row in np.asarray(f.near)}
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    of = oracle_replay(ip, ix, dv, P.block_sizes, P.tau, seg=owner, overrides=sorted(near))
    bst = np.concatenate([[0], np.cumsum(P.block_sizes)])
    worst, probs = 0.0, []
    for r, f in enumerate(exports):
        present = {int(bst[K]) for K in range(len(owner)) if owner[K] in (r, -1)}
        res = compare_present_blocks(f, of, present)
        worst = max(worst, res["max_rel"])
        probs += res["problems"][:2]
    out["parity_max_rel"] = worst
    out["parity_problems"] = probs
    xv = np.ones(P.n)
    want = np.empty(P.n)
    want[P.perm] = oracle.apply(of, xv[P.perm])
    out["apply_parity_max_rel"] = float(np.abs(y_dist.cpu().numpy() - want).max() / np.abs(want).max())
print(json.dumps(out), flush=True)
