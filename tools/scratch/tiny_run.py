import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from inputs.configs import random_dd, dense_to_csr
from paper_1908_10169_b200 import BILU
A = random_dd(40, 0.15, 1)
ip, ix, dv = dense_to_csr(A)
g = BILU(ip, ix, dv, [3, 5, 2, 4, 6, 1, 3, 8, 4, 4], aggregate=0, n_ctas=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
st = g.factor(1e-2)
print("ok", st["t_factor_ms"])
