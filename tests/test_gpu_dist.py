"""Distributed (multi-GPU) factorization path, checked on ONE GPU by running the ranks'
phases one after another in one process: every rank has its own context; phase A runs
for every rank, the packed interface buffers are handed over device-to-device (in place of
the NCCL all-gather, which tests/test_dist_gloo.py covers on CPU), then phase B runs for
every rank.  No kernel waits on another rank's kernel.  The union of the ranks' factors
must match the oracle run with the same aggregation segments (R18)."""
import numpy as np
import pytest

import oracle
from inputs.configs import config2, config5
from tests.parity import compare_present_blocks, oracle_replay

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1908_10169_b200.build import build
    build()


def run_simulated(P, world):
    from paper_1908_10169_b200 import BILU
    from paper_1908_10169_b200.dist import partition_owner
    owner = partition_owner(P.block_part, world)
    ctxs = [BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm) for _ in range(world)]
    for r, g in enumerate(ctxs):
        g.dist_setup(owner, r)
    for g in ctxs:
        g.factor_local(P.tau)
    bufs = [g.interface_pack() for g in ctxs]
    for r, g in enumerate(ctxs):
        for q in range(world):
            if q != r:
                g.interface_unpack(bufs[q])
    stats = [g.factor_separators() for g in ctxs]
    return owner, ctxs, stats, bufs


@pytest.mark.parametrize("world", [1, 2, 4])
def test_simulated_ranks_match_oracle_c5(world):
    P = config5(N=20, top_levels=2)          # 4 top-level subtrees, 3 separators
    owner, ctxs, stats, bufs = run_simulated(P, world)
    exports = [g.export() for g in ctxs]
    near = {tuple(int(x) for x in row) for f in exports for row in np.asarray(f.near)}
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    of = oracle_replay(ip, ix, dv, P.block_sizes, P.tau, seg=owner, overrides=sorted(near))
    bst = np.concatenate([[0], np.cumsum(P.block_sizes)])
    for r, f in enumerate(exports):
        present = {int(bst[K]) for K in range(len(owner)) if owner[K] in (r, -1)}
        res = compare_present_blocks(f, of, present)
        assert not res["problems"], (r, res["problems"][:3])
        assert res["checked"] > 0
    if world > 1:
        assert all(b.numel() > 0 for b in bufs)
    # the separator blocks are the same on every rank
    sep0 = {int(bst[K]) for K in range(len(owner)) if owner[K] == -1}
    for f in exports[1:]:
        assert not compare_present_blocks(f, exports[0], sep0, tol=1e-12)["problems"]


def test_simulated_ranks_c2_two_subtrees():
    P = config2(N=24, leaf=128, top_levels=1)
    owner, ctxs, stats, bufs = run_simulated(P, 2)
    exports = [g.export() for g in ctxs]
    near = {tuple(int(x) for x in row) for f in exports for row in np.asarray(f.near)}
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    of = oracle_replay(ip, ix, dv, P.block_sizes, P.tau, seg=owner, overrides=sorted(near))
    bst = np.concatenate([[0], np.cumsum(P.block_sizes)])
    for r, f in enumerate(exports):
        present = {int(bst[K]) for K in range(len(owner)) if owner[K] in (r, -1)}
        assert not compare_present_blocks(f, of, present)["problems"]


def test_dist_setup_rejects_non_separating_partition():
    from paper_1908_10169_b200 import BILU, BiluError
    P = config5(N=12, top_levels=1)
    g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
    bad = np.zeros(len(P.block_sizes), dtype=np.int32)
    bad[: len(bad) // 2] = 1            # cuts through coupled blocks
    with pytest.raises(BiluError):
        g.dist_setup(bad, 0)


def test_distributed_context_refuses_plain_calls():
    from paper_1908_10169_b200 import BILU, BiluError
    from paper_1908_10169_b200.dist import partition_owner
    P = config5(N=12, top_levels=1)
    g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
    g.dist_setup(partition_owner(P.block_part, 2), 0)
    with pytest.raises(BiluError):
        g.factor(P.tau)
    with pytest.raises(BiluError):
        g.interface_pack()            # before phase A


def test_simulated_ranks_c2_full_size_four_ranks():
    """BASELINE configs[1] at full size split over 4 simulated ranks (the bench's N=4 split)."""
    P = config2(top_levels=2)
    owner, ctxs, stats, bufs = run_simulated(P, 4)
    exports = [g.export() for g in ctxs]
    near = {tuple(int(x) for x in row) for f in exports for row in np.asarray(f.near)}
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    of = oracle_replay(ip, ix, dv, P.block_sizes, P.tau, seg=owner, overrides=sorted(near))
    bst = np.concatenate([[0], np.cumsum(P.block_sizes)])
    for r, f in enumerate(exports):
        present = {int(bst[K]) for K in range(len(owner)) if owner[K] in (r, -1)}
        res = compare_present_blocks(f, of, present)
        assert not res["problems"], (r, res["problems"][:3])


def _dist_apply_simulated(ctxs, x):
    """bilu_apply_dist_begin on every rank, the sum of the contributions (the all-reduce),
    bilu_apply_dist_end on every rank (separators written by rank 0), the sum of the shares."""
    contribs = [g.apply_dist_begin(x) for g in ctxs]
    total = sum(c.clone() for c in contribs) if contribs[0].numel() else contribs[0]
    ys = [g.apply_dist_end(total, write_separators=(r == 0)) for r, g in enumerate(ctxs)]
    return sum(ys)


@pytest.mark.parametrize("world", [1, 2, 4])
def test_distributed_apply_matches_oracle_c5(world):
    """NEXT-1 multi-GPU apply: the ranks' two-phase sweeps give the oracle's M^{-1} x for the
    factorization with the same segments."""
    import torch
    P = config5(N=20, top_levels=2)
    owner, ctxs, stats, bufs = run_simulated(P, world)
    exports = [g.export() for g in ctxs]
    near = {tuple(int(x) for x in row) for f in exports for row in np.asarray(f.near)}
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    of = oracle_replay(ip, ix, dv, P.block_sizes, P.tau, seg=owner, overrides=sorted(near))
    rng = np.random.default_rng(world)
    for xv in (np.ones(P.n), rng.standard_normal(P.n)):
        y = _dist_apply_simulated(ctxs, torch.tensor(xv, device="cuda")).cpu().numpy()
        yp = oracle.apply(of, xv[P.perm])
        want = np.empty(P.n)
        want[P.perm] = yp
        err = np.abs(y - want).max() / np.abs(want).max()
        assert err < 1e-10, err
    for g in ctxs:       # the single-context apply refuses distributed factors
        from paper_1908_10169_b200 import BiluError
        with pytest.raises(BiluError):
            g.apply(0, 0)


def test_distributed_apply_c2_two_subtrees():
    import torch
    P = config2(N=24, leaf=128, top_levels=1)
    owner, ctxs, stats, bufs = run_simulated(P, 2)
    exports = [g.export() for g in ctxs]
    near = {tuple(int(x) for x in row) for f in exports for row in np.asarray(f.near)}
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    of = oracle_replay(ip, ix, dv, P.block_sizes, P.tau, seg=owner, overrides=sorted(near))
    xv = np.random.default_rng(7).standard_normal(P.n)
    y = _dist_apply_simulated(ctxs, torch.tensor(xv, device="cuda")).cpu().numpy()
    want = np.empty(P.n)
    want[P.perm] = oracle.apply(of, xv[P.perm])
    assert np.abs(y - want).max() / np.abs(want).max() < 1e-10


def test_distributed_apply_order_errors():
    import torch
    from paper_1908_10169_b200 import BiluError
    P = config5(N=12, top_levels=1)
    owner, ctxs, stats, bufs = run_simulated(P, 2)
    with pytest.raises(BiluError):       # end before begin
        ctxs[0].apply_dist_end(torch.zeros(max(1, P.n), dtype=torch.float64, device="cuda"), True)
