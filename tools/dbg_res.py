import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NFFTK_TILE"] = "8"
import numpy as np
import paper_1810_09891_b200 as nf
from oracle import oracle as O

def e2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(a))

m = int(sys.argv[1]) if len(sys.argv) > 1 else 6
N, n = (8, 8, 8), (32, 32, 32)
rng = np.random.default_rng(0)
for trial, M in enumerate([1, 1, 1, 2, 5, 40, 300, 3000]):
    x = rng.random((M, 3)) - 0.5
    fs = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    p = nf.Plan(N, M, n=n, m=m)
    p.x = x
    p.precompute()
    a = p.adjoint(fs)
    r = O.adjoint(N, n, m, x, fs)
    cells = np.floor(x * 32).astype(int) % 8
    print(M, p.gridding, e2(r, a), cells[:3].tolist())
