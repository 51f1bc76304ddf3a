"""Run trafo + adjoint of one BASELINE config a few times (for ncu / nsys-free
profiling).  Usage: python tools/profile_config.py C5 [reps] [--psi direct|tensor]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1810_09891_b200 as nf  # noqa: E402
from paper_1810_09891_b200 import workloads as wl  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2
    psi = None
    if "--psi" in sys.argv:
        psi = sys.argv[sys.argv.index("--psi") + 1]
    prec = "single" if "--single" in sys.argv else "double"
    w = wl.lookup(name)
    p = nf.Plan(w.N, w.M, n=w.n, m=w.m, precision=prec)
    if psi:
        p.set_psi_policy(nf.MODE_DIRECT if psi == "direct" else nf.MODE_TENSOR)
    p.x = torch.from_numpy(wl.nodes(w)).cuda()
    p.precompute()
    cdt = torch.complex64 if prec == "single" else torch.complex128
    fh = torch.from_numpy(wl.fhat(w)).cuda().to(cdt)
    fs = torch.from_numpy(wl.samples(w)).cuda().to(cdt)
    for _ in range(reps):
        p.trafo(fh)
        p.adjoint(fs)
    torch.cuda.synchronize()
    print("ok", name, p.tile, p._params()[10:12])


if __name__ == "__main__":
    main()
