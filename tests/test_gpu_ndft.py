"""Exact sums on the GPU (Plan.ndft / Plan.ndft_adjoint, csrc/ndft.cu) against
the reference's own ndft vectors (tests/golden, produced by transform.py:188-234)
and the CPU oracle, including d = 4 (the reference's einsum path) and the
chunked ZGEMM path at a config size."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_1810_09891_b200 as nf
from paper_1810_09891_b200 import workloads as wl

pytestmark = pytest.mark.gpu

SMALL = np.load(os.path.join(GOLDEN, "small_cases.npz"))
NAMES = sorted({k.split("__")[0] for k in SMALL.files})
TOL = 1e-12


def e2(ref, got):
    ref = np.asarray(ref).astype(np.complex128).ravel()
    got = np.asarray(got).astype(np.complex128).ravel()
    return float(np.linalg.norm(ref - got) / np.linalg.norm(ref))


def plan_with_nodes(N, x, **kw):
    p = nf.Plan(tuple(int(v) for v in N), x.shape[0], **kw)
    p.x = x
    return p


@pytest.mark.parametrize("name", NAMES)
def test_ndft_vs_reference_goldens(name):
    N, x = SMALL[f"{name}__N"], SMALL[f"{name}__x"]
    p = plan_with_nodes(N, x, n=tuple(int(v) for v in SMALL[f"{name}__n"]), m=int(SMALL[f"{name}__m"]))
    assert e2(SMALL[f"{name}__ndft"], p.ndft(SMALL[f"{name}__fhat"])) < TOL
    assert e2(SMALL[f"{name}__ndft_adjoint"], p.ndft_adjoint(SMALL[f"{name}__f"])) < TOL
    # module-level entry points of the reference (transform.ndft / ndft_adjoint)
    assert np.array_equal(nf.ndft(p, SMALL[f"{name}__fhat"]), p.ndft(SMALL[f"{name}__fhat"]))


def direct_sums(N, x, fh, f):
    """Small d = 4 restatement of transform.py:188-234 (the C oracle stops
    at d = 3): full phase matrix over the index set, k = -N/2 .. N/2-1."""
    ks = np.stack(np.meshgrid(*[np.arange(-(n // 2), n - n // 2) for n in N], indexing="ij"),
                  axis=-1).reshape(-1, len(N))
    ph = np.exp(-2j * np.pi * (ks @ x.T))  # (|I_N|, M)
    return ph.T @ fh, ph.conj() @ f


def test_ndft_d4_vs_direct_sums():
    rng = np.random.default_rng(4)
    N = (4, 6, 4, 2)
    x = rng.random((97, 4)) - 0.5
    fh = rng.standard_normal(int(np.prod(N))) + 1j * rng.standard_normal(int(np.prod(N)))
    f = rng.standard_normal(97) + 1j * rng.standard_normal(97)
    p = plan_with_nodes(N, x, n=(8, 12, 8, 4), m=1)
    ref_f, ref_a = direct_sums(N, x, fh, f)
    assert e2(ref_f, p.ndft(fh)) < TOL
    assert e2(ref_a, p.ndft_adjoint(f)) < TOL


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_ndft_configs_vs_oracle(cfg, oracle):
    w = wl.CONFIGS[cfg]
    x, fh, fs = wl.nodes(w), wl.fhat(w), wl.samples(w)
    p = plan_with_nodes(w.N, x, n=w.n, m=w.m)
    assert e2(oracle.ndft(w.N, x, fh), p.ndft(fh)) < TOL
    assert e2(oracle.ndft_adjoint(w.N, x, fs), p.ndft_adjoint(fs)) < TOL


def test_ndft_chunked_c3_subsample(oracle):
    """C3 (M = 262144, |I_N| = 64^3): several node chunks of the ZGEMM path;
    the forward sums checked on an oracle subsample, the adjoint through the
    identity <ndft(fhat), f> = <fhat, ndft_adjoint(f)>."""
    w = wl.CONFIGS["C3"]
    x, fh, fs = wl.nodes(w), wl.fhat(w), wl.samples(w)
    p = plan_with_nodes(w.N, x, n=w.n, m=w.m)
    f = p.ndft(fh)
    idx = np.random.default_rng(0).choice(w.M, 512, replace=False)
    assert e2(oracle.ndft(w.N, x[idx], fh), f[idx]) < TOL
    a = p.ndft_adjoint(fs)
    lhs, rhs = np.vdot(fs, f), np.vdot(a, fh)
    assert abs(lhs - rhs) <= 1e-11 * abs(lhs)


def test_ndft_device_tensors_match_host():
    import torch

    name = "d3_m6"
    N, x = SMALL[f"{name}__N"], SMALL[f"{name}__x"]
    p = plan_with_nodes(N, x, n=tuple(int(v) for v in SMALL[f"{name}__n"]))
    fh = SMALL[f"{name}__fhat"]
    got = p.ndft(torch.from_numpy(fh).cuda())
    assert got.is_cuda and got.dtype == torch.complex128
    assert np.array_equal(got.cpu().numpy(), p.ndft(fh))


def test_ndft_errors():
    p = nf.Plan((8, 8), 10)
    with pytest.raises(nf.PlanStateError):
        p.ndft(np.zeros(64, complex))
    p.x = np.zeros((10, 2))
    with pytest.raises(nf.ShapeError):
        p.ndft(np.zeros(63, complex))
    with pytest.raises(nf.ShapeError):
        p.ndft_adjoint(np.zeros(11, complex))
