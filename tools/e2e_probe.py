"""Time each reference C-ABI call of the e2e step (C3) separately."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_09891_b200 import _lib  # noqa: E402
from paper_1810_09891_b200 import workloads as wl  # noqa: E402

w = wl.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
lib = _lib.load()
h = lib.nfftk_create_advanced(_lib.i32_array(w.N), w.d, w.M, _lib.i32_array(w.n), w.m, 0x1fd1, 0x41)
x = np.ascontiguousarray(wl.nodes(w))
assert lib.nfftk_set_x(h, x.ctypes.data, x.size) == 0
fh = np.ascontiguousarray(wl.fhat(w)).view(np.float64)
fs = np.ascontiguousarray(wl.samples(w)).view(np.float64)
names = ["set_fhat", "trafo", "set_f", "adjoint"]
calls = [lambda: lib.nfftk_set_fhat(h, fh.ctypes.data, fh.size), lambda: lib.nfftk_trafo(h),
         lambda: lib.nfftk_set_f(h, fs.ctypes.data, fs.size), lambda: lib.nfftk_adjoint(h)]
acc = {n: 0.0 for n in names}
for it in range(13):
    for n, c in zip(names, calls):
        t0 = time.perf_counter()
        assert c() == 0
        dt = time.perf_counter() - t0
        if it >= 3:
            acc[n] += dt
print({n: round(v / 10 * 1e3, 4) for n, v in acc.items()}, "ms")
