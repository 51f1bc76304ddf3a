"""Small plans through every new kernel path (adjoint-identity sanity check; also the
driver for compute-sanitizer where the pool allows it):
   compute-sanitizer --tool memcheck|racecheck python tools/sanitize_small.py
(pruned FFT d=2 / d=3 incl. long lines and both line groups, gathering spreads:
residue, d=2 one / two warps, d=3 rows; complex128 and complex64)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_09891_b200 as nf  # noqa: E402

rng = np.random.default_rng(0)
CASES = [((16, 16, 16), (32, 32, 32), 4, 6000, None),      # residue spread (8^3 tiles), cuFFT (n = 32)
         ((32, 32, 32), (64, 64, 64), 4, 20000, None),     # residue + pruned FFT
         ((32, 32, 32), (64, 64, 64), 6, 3000, None),      # row spread + pruned FFT
         ((32, 64), (64, 128), 6, 3000, None),             # d=2 spread + pruned FFT
         ((512, 8), (1024, 64), 4, 2000, None),            # long lines
         ((8, 1024), (64, 2048), 4, 2000, None)]
for prec in ("double", "single"):
    for N, n, m, M, _ in CASES:
        x = rng.random((M, len(N))) - 0.5
        x[0] = -0.5
        K = int(np.prod(N))
        fh = rng.standard_normal(K) + 1j * rng.standard_normal(K)
        fs = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        p = nf.Plan(N, M, n=n, m=m, precision=prec)
        p.x = x
        p.precompute()
        f = p.trafo(fh)
        a = p.adjoint(fs)
        # adjoint identity as a sanity check
        lhs = np.vdot(np.asarray(f, np.complex128), fs)
        rhs = np.vdot(fh, np.asarray(a, np.complex128))
        rel = abs(lhs - rhs) / abs(lhs)
        print(prec, N, n, m, p.gridding, p.fft, "identity %.2e" % rel)
        assert rel < (1e-10 if prec == "double" else 1e-4)
        p.close()
print("done")
