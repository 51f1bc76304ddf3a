"""Full-size parity at the BASELINE configurations C3, C4 and C5, trafo AND
adjoint, complex128 and complex64.

The goldens (``tests/golden/C{3,4,5}_full.npz``) come from running the LIVE
reference ``nfftk.Plan`` (default flags, /root/reference/pkg/src/nfftk/
transform.py:92-176) at each configuration's full size in the build
container (``tests/golden/make_golden.py C3 C4 C5``).  Each stores 65,536
seeded entries of the trafo output f and of the adjoint output f_hat, plus
whole-vector norms, sums and 4,096 block sums -- so the device run is checked
entry-wise on the subsample AND over the whole vector (block sums localise a
wrong region anywhere in it).

Tolerances (BASELINE.json north_star): relative l2 <= 1e-12 for complex128,
<= 1e-5 for complex64 (the reference has no complex64 path; its complex128
output is the oracle).  The C4 adjoint is also compared as a whole vector
against the oracle's C port of the reference path.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_1810_09891_b200 as nf
from paper_1810_09891_b200 import workloads as wl

pytestmark = pytest.mark.gpu

TOL = {"double": 1e-12, "single": 1e-5}
BLOCKS = 4096


def rel(ref, got):
    ref = np.asarray(ref).astype(np.complex128).ravel()
    got = np.asarray(got).astype(np.complex128).ravel()
    return float(np.linalg.norm(ref - got) / np.linalg.norm(ref))


def block_sums(v, blocks=BLOCKS):
    """Same slicing as make_golden.block_sums, on the device (fp64 sums)."""
    import torch

    n = v.numel()
    edges = (torch.arange(blocks + 1, dtype=torch.int64) * n) // blocks
    sizes = (edges[1:] - edges[:-1]).to(v.device)
    seg = torch.repeat_interleave(torch.arange(blocks, device=v.device), sizes)
    out = torch.zeros(blocks, dtype=torch.complex128, device=v.device)
    out.index_add_(0, seg, v.to(torch.complex128))
    return out.cpu().numpy()


_RUNS = {}


def run_config(cfg, precision):
    """trafo and adjoint of the whole configuration on the GPU (cached per
    (cfg, precision): several tests inspect the same run; the outputs of all
    six runs together are < 3 GiB of device memory)."""
    key = (cfg, precision)
    if key in _RUNS:
        return _RUNS[key]
    import torch

    torch.cuda.empty_cache()
    w = wl.CONFIGS[cfg]
    dev = torch.device("cuda", 0)
    cdt = torch.complex64 if precision == "single" else torch.complex128
    p = nf.Plan(w.N, w.M, n=w.n, m=w.m, precision=precision)
    p.x = torch.from_numpy(wl.nodes(w)).to(dev)
    p.precompute()
    f = p.trafo(torch.from_numpy(wl.fhat(w)).to(dev, cdt))
    a = p.adjoint(torch.from_numpy(wl.samples(w)).to(dev, cdt))
    torch.cuda.synchronize()
    p.close()
    _RUNS[key] = (w, f, a)
    return _RUNS[key]


CASES = [(c, prec) for c in ("C3", "C4", "C5") for prec in ("double", "single")]


@pytest.mark.parametrize("cfg,precision", CASES)
def test_fullsize_trafo_vs_reference(cfg, precision):
    import torch

    g = np.load(os.path.join(GOLDEN, f"{cfg}_full.npz"))
    w, f, _ = run_config(cfg, precision)
    tol = TOL[precision]
    idx = torch.from_numpy(g["trafo_idx"]).to(f.device)
    assert rel(g["trafo_sub"], f[idx].cpu().numpy()) < tol
    # whole vector: norm, block sums, sum
    nrm = torch.linalg.norm(f.to(torch.complex128)).item()
    assert abs(nrm - float(g["norm_f"])) / float(g["norm_f"]) < tol
    assert rel(g["blocksum_f"], block_sums(f)) < tol
    s = f.to(torch.complex128).sum().item()
    assert abs(s - complex(g["sum_f"])) < tol * np.sqrt(w.M) * float(g["norm_f"])


@pytest.mark.parametrize("cfg,precision", CASES)
def test_fullsize_adjoint_vs_reference(cfg, precision):
    import torch

    g = np.load(os.path.join(GOLDEN, f"{cfg}_full.npz"))
    w, _, a = run_config(cfg, precision)
    tol = TOL[precision]
    idx = torch.from_numpy(g["adjoint_idx"]).to(a.device)
    assert rel(g["adjoint_sub"], a[idx].cpu().numpy()) < tol
    nrm = torch.linalg.norm(a.to(torch.complex128)).item()
    assert abs(nrm - float(g["norm_fhat"])) / float(g["norm_fhat"]) < tol
    assert rel(g["blocksum_fhat"], block_sums(a)) < tol
    s = a.to(torch.complex128).sum().item()
    assert abs(s - complex(g["sum_fhat"])) < tol * np.sqrt(w.num_freqs) * float(g["norm_fhat"])


@pytest.mark.parametrize("precision", ["double", "single"])
def test_c4_full_adjoint_vs_oracle(precision, oracle):
    """The clustered C4 adjoint (the spreading-contention config) as a whole
    |I_N| vector against the oracle's C port of the reference adjoint."""
    w, _, a = run_config("C4", precision)
    ref = oracle.adjoint(w.N, w.n, w.m, wl.nodes(w), wl.samples(w))
    assert rel(ref, a.cpu().numpy()) < TOL[precision]


def test_c4_full_trafo_vs_oracle(oracle):
    w, f, _ = run_config("C4", "double")
    ref = oracle.trafo(w.N, w.n, w.m, wl.nodes(w), wl.fhat(w))
    assert rel(ref, f.cpu().numpy()) < TOL["double"]
