"""Host logic of the multi-GPU path on CPU (world_size 2, gloo): the variable-size
all-gather used for the interface exchange, and the subtree -> rank assignment."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_10169_b200.dist import exchange_variable
    local = torch.full(((rank + 1) * 1000 + 3,), rank + 7, dtype=torch.uint8)
    bufs = exchange_variable(local)
    res = [(int(b.numel()), int(b.min()), int(b.max())) for b in bufs]
    # an empty contribution from one rank
    local2 = torch.zeros(0 if rank == 0 else 5, dtype=torch.uint8)
    bufs2 = exchange_variable(local2)
    res2 = [int(b.numel()) for b in bufs2]
    out.put((rank, res, res2))
    dist.destroy_process_group()


def test_exchange_variable_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, res, res2 in got:
        assert res == [(1003, 7, 7), (2003, 8, 8)]
        assert res2 == [0, 5]


def test_partition_owner():
    from paper_1908_10169_b200.dist import partition_owner
    part = np.array([0, 0, 1, 1, -1, 2, 3, -1, -1])
    assert partition_owner(part, 1).tolist() == [0, 0, 0, 0, -1, 0, 0, -1, -1]
    assert partition_owner(part, 2).tolist() == [0, 0, 0, 0, -1, 1, 1, -1, -1]
    assert partition_owner(part, 4).tolist() == [0, 0, 1, 1, -1, 2, 3, -1, -1]
    with pytest.raises(ValueError):
        partition_owner(part, 8)


def test_partition_of_nd_orderings_separates():
    """The ND generator's subtree labels give a partition with no coupling across ranks
    and no subtree block after a separator it touches (what bilu_dist_setup checks)."""
    import scipy.sparse as sp
    from inputs.configs import config5
    from paper_1908_10169_b200.dist import partition_owner
    P = config5(N=16, top_levels=2)
    assert len(np.unique(P.block_part[P.block_part >= 0])) == 4
    owner = partition_owner(P.block_part, 4)
    bst = np.concatenate([[0], np.cumsum(P.block_sizes)])
    blk = np.repeat(np.arange(len(P.block_sizes)), P.block_sizes)
    inv = np.empty(P.n, dtype=np.int64); inv[P.perm] = np.arange(P.n)
    A = sp.csr_matrix((P.data, P.indices, P.indptr), shape=(P.n, P.n)).tocoo()
    bi, bj = blk[inv[A.row]], blk[inv[A.col]]
    a, b = np.minimum(bi, bj), np.maximum(bi, bj)
    oa, ob = owner[a], owner[b]
    assert not np.any((oa >= 0) & (ob >= 0) & (oa != ob))
    assert not np.any((oa == -1) & (ob >= 0) & (a != b))


class _FakeRankCtx:
    """Stands in for a rank's BILU context on CPU: a 6-row problem, rows 0-1 owned by rank 0,
    rows 2-3 by rank 1, rows 4-5 separators.  begin returns rank-specific contributions; end
    checks it received their sum and returns its share of y."""
    def __init__(self, rank):
        self.rank = rank
        self.n = 6

    def apply_dist_begin(self, x):
        import torch
        return torch.tensor([1.0 + self.rank, 10.0 * (self.rank + 1)], dtype=torch.float64) + x[4:6]

    def apply_dist_end(self, s, write_separators):
        import torch
        self.got = s.clone()
        y = torch.zeros(6, dtype=torch.float64)
        own = slice(0, 2) if self.rank == 0 else slice(2, 4)
        y[own] = float(self.rank + 1)
        if write_separators:
            y[4:6] = s
        return y


def _apply_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_10169_b200.dist import apply_distributed
    g = _FakeRankCtx(rank)
    x = torch.arange(6, dtype=torch.float64)
    y = apply_distributed(g, x)
    out.put((rank, g.got.tolist(), y.tolist()))
    dist.destroy_process_group()


def test_apply_distributed_gloo_world2():
    """apply_distributed: one all-reduce of the separator contributions (every rank gets the
    sum), disjoint shares of y (separators from rank 0 only) summed into the full vector."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_apply_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    s = [1.0 + 2.0 + 4 + 4, 10.0 + 20.0 + 5 + 5]
    for rank, recv, y in got:
        assert recv == s
        assert y == [1.0, 1.0, 2.0, 2.0] + s
