"""Kernel A/B timing with a parity check: python tools/kbench.py C5 [--single] [--reps 10]

Builds one plan on the configuration's seeded nodes (device), checks trafo and
adjoint against the committed full-size reference goldens (tests/golden/
<C>_full.npz, 65,536 seeded entries each), then times `reps` trafo+adjoint
pairs with the library's per-phase CUDA events.  NFFTK_LIB selects an A/B
build (tools/build_variant.sh).  Prints one line per run."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_09891_b200 as nf  # noqa: E402
from paper_1810_09891_b200 import workloads as wl  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    return float(np.linalg.norm(a - b) / np.linalg.norm(a))


def main():
    name = sys.argv[1]
    single = "--single" in sys.argv
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 10
    w = wl.lookup(name)
    prec = "single" if single else "double"
    cdt = torch.complex64 if single else torch.complex128
    p = nf.Plan(w.N, w.M, n=w.n, m=w.m, precision=prec)
    p.x = torch.from_numpy(wl.nodes(w)).cuda()
    p.precompute()
    fh = torch.from_numpy(wl.fhat(w)).cuda().to(cdt)
    fs = torch.from_numpy(wl.samples(w)).cuda().to(cdt)
    f = p.trafo(fh)
    a = p.adjoint(fs)
    g = os.path.join(ROOT, "tests", "golden", f"{name}_full.npz")
    err = {}
    if os.path.exists(g):
        G = np.load(g)
        err["trafo"] = rel(G["trafo_sub"], f[torch.from_numpy(G["trafo_idx"]).cuda()].cpu().numpy())
        err["adjoint"] = rel(G["adjoint_sub"], a[torch.from_numpy(G["adjoint_idx"]).cuda()].cpu().numpy())
    for _ in range(3):
        p.trafo(fh, out=f)
        p.adjoint(fs, out=a)
    torch.cuda.synchronize()
    p.phase_times(reset=True)
    p.set_timing(True)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(reps):
        p.trafo(fh, out=f)
        p.adjoint(fs, out=a)
    s1.record()
    torch.cuda.synchronize()
    ph = {k: v[0] / reps for k, v in p.phase_times(reset=True).items() if v[1]}
    out = {"config": name, "prec": prec, "lib": os.environ.get("NFFTK_LIB", "in-tree"),
           "step_ms": s0.elapsed_time(s1) / reps, "err": err,
           "interp": ph.get("interp"), "spread": ph.get("spread"),
           "phases": {k: round(v, 4) for k, v in ph.items()}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
