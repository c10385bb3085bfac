"""The distributed factorization and apply across real
processes: two ranks, each its own process, torch.distributed process group and library
context (gloo transport; one GPU here, so both contexts live on cuda:0 -- no kernel waits
on another rank's kernel, the exchange is host-level).  The union of the ranks' factors
must match the oracle run with the same aggregation segments (R18), and the
ranks' M^{-1} x the oracle's (L P U)^{-1} x."""
import multiprocessing as mp
import pickle
import socket

import numpy as np
import pytest

import oracle
from inputs.configs import config2, config5
from tests.parity import compare_present_blocks, oracle_replay

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, cfg, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1908_10169_b200.build import build
    build()
    from tests.dist_worker import worker
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, str(tmp_path), cfg)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    codes = [p.exitcode for p in procs]
    for p in procs:
        if p.is_alive():
            p.kill()
    assert codes == [0] * world, codes
    return [pickle.load(open(tmp_path / ("rank%d.pkl" % r), "rb")) for r in range(world)]


@pytest.mark.parametrize("world,cfg", [
    (2, ("c2", dict(N=24, leaf=128, top_levels=1))),
    (2, ("c5", dict(N=20, top_levels=2))),
    (4, ("c5", dict(N=20, top_levels=2))),
])
def test_processes_match_oracle(world, cfg, tmp_path):
    outs = _run(world, cfg, tmp_path)
    name, kw = cfg
    P = (config2 if name == "c2" else config5)(**kw)
    owner = outs[0]["owner"]
    near = {tuple(int(x) for x in row) for o in outs for row in np.asarray(o["factor"].near)}
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    of = oracle_replay(ip, ix, dv, P.block_sizes, P.tau, seg=owner, overrides=sorted(near))
    bst = np.concatenate([[0], np.cumsum(P.block_sizes)])
    for r, o in enumerate(outs):
        assert o["sent"] > 0 and o["recv"] > 0
        present = {int(bst[K]) for K in range(len(owner)) if owner[K] in (r, -1)}
        res = compare_present_blocks(o["factor"], of, present)
        assert not res["problems"], (r, res["problems"][:3])
        assert res["checked"] > 0
    # every rank ends with the same y = M^{-1} x (assembled by the second all-reduce)
    xv = outs[0]["x"]
    want = np.empty(P.n)
    want[P.perm] = oracle.apply(of, xv[P.perm])
    for o in outs:
        err = np.abs(o["y"] - want).max() / np.abs(want).max()
        assert err < 1e-10, err
