"""One device ILU(1,tau) estimate and one cosine blocking of a config (for ncu launch lists).
python tools/blocking_probe.py c5"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs.configs import make_config  # noqa: E402
from paper_1908_10169_b200 import cosine_blocks, ilu1_blocks  # noqa: E402

P = make_config(sys.argv[1] if len(sys.argv) > 1 else "c5")
bs, nl = ilu1_blocks(P.indptr, P.indices, P.data, P.tau, 8, perm=P.perm)
q, cs, cl = cosine_blocks(P.indptr, P.indices, 0.8, 128)
print("ilu1 blocks", len(bs), "launches", nl, "| cosine groups", len(cs), "launches", cl)
