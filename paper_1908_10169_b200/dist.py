"""Multi-GPU factorization over nested-dissection subtrees.

One process per GPU.  Every rank holds the same global matrix, ordering and initial
partition; the top-level ND subtrees are assigned to ranks (`partition_owner`), then

  phase A   bilu_factor_local       each rank factors its own subtrees -- no communication
                                    (inside an ND subtree every contributor is a block of
                                    the same subtree)
  exchange  exchange_variable       the ranks' packed interface panels (the kept L rows /
                                    Ũ columns of subtree blocks in separator rows / columns:
                                    the operands of the separator Schur updates) are
                                    all-gathered: sizes by all_gather, payloads by one
                                    broadcast per rank (NCCL over NVLink on GPUs, gloo on CPU)
  phase B   bilu_factor_separators  every rank factors the separator blocks (replicated),
                                    then aggregates within its own blocks

The preconditioner is applied the same way (`apply_distributed`): forward sweep over the
own subtrees, one all-reduce of the separator-row contributions, the separator sweeps
(replicated) and the backward sweep over own subtree blocks, one all-reduce assembling y.

torch.distributed is the transport only (plumbing); every arithmetic step runs in the
library's kernels.
"""
from __future__ import annotations

import numpy as np


def partition_owner(block_part, world: int) -> np.ndarray:
    """Owner rank of every initial block: top-level subtree s of n_sub goes to rank
    s * world // n_sub (contiguous groups); separator blocks (part -1) -> -1."""
    part = np.asarray(block_part, dtype=np.int64)
    sub = part[part >= 0]
    n_sub = int(sub.max()) + 1 if len(sub) else 1
    if world > n_sub:
        raise ValueError("world size %d exceeds the %d top-level subtrees" % (world, n_sub))
    owner = np.where(part >= 0, (part * world) // n_sub, -1)
    return owner.astype(np.int32)


def exchange_variable(local, group=None):
    """All-gather of one variable-size uint8 tensor per rank (CUDA tensors with NCCL, CPU
    tensors with gloo).  Returns the list of every rank's tensor (this rank's is `local`)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    if local.is_cuda and dist.get_backend(group) == "gloo":
        # gloo moves CPU tensors only (all_gather): stage the payloads through host memory
        return [b.to(local.device) if r != me else local
                for r, b in enumerate(exchange_variable(local.cpu(), group))]
    n = torch.tensor([local.numel()], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    out = []
    for r in range(world):
        if r == me:
            buf = local
        else:
            buf = torch.empty(int(sizes[r].item()), dtype=torch.uint8, device=local.device)
        src = dist.get_global_rank(group, r) if group is not None else r
        dist.broadcast(buf, src=src, group=group)
        out.append(buf)
    return out


def factor_distributed(g, tau, group=None, timer=None):
    """Phase A, exchange, phase B on this rank's context `g` (a BILU set up with
    dist_setup).  `timer(name)` (optional) is called after each step for device timing.
    Returns (stats, bytes sent, bytes received)."""
    import torch.distributed as dist
    me = dist.get_rank(group)
    g.local_stats = g.factor_local(tau)
    if timer:
        timer("local")
    mine = g.interface_pack()
    bufs = exchange_variable(mine, group)
    if timer:
        timer("exchange")
    recv = 0
    for r, b in enumerate(bufs):
        if r != me:
            g.interface_unpack(b)
            recv += b.numel()
    st = g.factor_separators()
    if timer:
        timer("separators")
    return st, int(mine.numel()), recv


def apply_distributed(g, x, group=None):
    """y = M^{-1} x with the ranks' distributed factors (`g` after factor_distributed; x the
    same CUDA float64 vector on every rank).  Two all-reduces: the separator contributions of
    the forward sweep, and the assembly of y from the ranks' disjoint shares."""
    import torch.distributed as dist
    contrib = g.apply_dist_begin(x)
    _all_reduce(contrib, group)
    y = g.apply_dist_end(contrib, write_separators=dist.get_rank(group) == 0)
    _all_reduce(y, group)
    return y


def _all_reduce(t, group=None):
    """Sum over the ranks in place (NCCL on CUDA tensors; gloo stages through host memory)."""
    import torch.distributed as dist
    if t.is_cuda and dist.get_backend(group) == "gloo":
        h = t.cpu()
        dist.all_reduce(h, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, group=group)
