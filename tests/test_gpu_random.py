"""Seeded random plans against the CPU oracle: d = 3 grids around the tile and
halo sizes (partial tiles, n barely above the halo), anisotropic shapes, every
cutoff, both precisions, uniform / clustered / grid-aligned node mixes and
node counts from a handful to dense tiles -- whichever gridding kernels the
plan picks (batch, pipelined rows, residue-owned spread)."""

import numpy as np
import pytest

import paper_1810_09891_b200 as nf

pytestmark = pytest.mark.gpu

TOL = {"double": 1e-12, "single": 2e-5}


def e2(ref, got):
    ref = np.asarray(ref).astype(np.complex128).ravel()
    got = np.asarray(got).astype(np.complex128).ravel()
    return float(np.linalg.norm(ref - got) / np.linalg.norm(ref))


def draw(seed):
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(1, 7))
    n = tuple(int(2 * rng.integers((2 * m + 10) // 2, 26)) for _ in range(3))
    N = tuple(int(2 * rng.integers(1, max(2, ni // 4))) for ni in n)
    M = int(rng.choice([3, 40, 700, 6000, 25000]))
    kind = rng.choice(["uniform", "clustered", "aligned"])
    x = rng.random((M, 3)) - 0.5
    if kind == "clustered":
        c = rng.random((3, 3)) - 0.5
        x = (c[rng.integers(0, 3, M)] + 0.02 * rng.standard_normal((M, 3)) + 0.5) % 1.0 - 0.5
    elif kind == "aligned":
        k = max(1, M // 3)
        x[:k] = rng.integers(-8, 8, size=(k, 3)) / np.array(n)
        x[k:2 * k, int(rng.integers(0, 3))] = -0.5
    precision = "single" if seed % 3 == 0 else "double"
    tile = int(rng.choice([0, 8, 8]))
    return N, n, m, np.ascontiguousarray(np.clip(x, -0.5, np.nextafter(0.5, 0))), precision, tile


@pytest.mark.parametrize("seed", range(36))
def test_random_plan(seed, oracle, monkeypatch):
    N, n, m, x, precision, tile = draw(seed)
    if tile:
        monkeypatch.setenv("NFFTK_TILE", str(tile))
    else:
        monkeypatch.delenv("NFFTK_TILE", raising=False)
    rng = np.random.default_rng(seed)
    K, M = int(np.prod(N)), x.shape[0]
    fh = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    fs = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    p = nf.Plan(N, M, n=n, m=m, precision=precision)
    p.x = x
    p.precompute()
    for _ in range(2):
        assert e2(oracle.trafo(N, n, m, x, fh), p.trafo(fh)) < TOL[precision], (N, n, m, M, precision, p.gridding)
        assert e2(oracle.adjoint(N, n, m, x, fs), p.adjoint(fs)) < TOL[precision], (N, n, m, M, precision, p.gridding)
    p.close()
