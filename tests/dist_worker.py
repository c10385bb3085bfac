"""One rank of a real multi-process run of the distributed factorization,
used by tests/test_gpu_dist_procs.py.  Every rank is its own process with its own
torch.distributed rank (gloo: on one GPU NCCL refuses two ranks per device) and its own
library context on cuda:0; the ranks' kernels never wait on one another -- the only
cross-rank steps are the host-level collectives of dist.factor_distributed /
dist.apply_distributed.  The rank writes its exported factors and M^{-1} x to `outdir`."""
import os
import pickle
import sys


def worker(rank, world, port, outdir, cfg):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import numpy as np
    import torch
    import torch.distributed as dist
    from inputs.configs import config2, config5
    from paper_1908_10169_b200 import BILU
    from paper_1908_10169_b200.dist import apply_distributed, factor_distributed, partition_owner

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        name, kw = cfg
        P = (config2 if name == "c2" else config5)(**kw)
        torch.cuda.set_device(0)
        g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
        owner = partition_owner(P.block_part, world)
        g.dist_setup(owner, rank)
        st, sent, recv = factor_distributed(g, P.tau)
        x = torch.tensor(np.random.default_rng(11).standard_normal(P.n), device="cuda")
        y = apply_distributed(g, x)
        out = {"owner": owner, "factor": g.export(), "y": y.cpu().numpy(), "x": x.cpu().numpy(),
               "sent": sent, "recv": recv, "n_blocks_final": int(st["n_blocks_final"])}
        with open(os.path.join(outdir, "rank%d.pkl" % rank), "wb") as f:
            pickle.dump(out, f)
        g.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()
