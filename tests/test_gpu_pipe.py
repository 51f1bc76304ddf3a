"""Parity of the pipelined register kernels (k_interp_pipe, k_spread_pipe,
k_spread2_pipe) against the CPU oracle on their own tile geometries:
d=3 with 8^3 tiles (forced with NFFTK_TILE on small grids), d=2 with 32-row
halos, every cutoff they are instantiated for, complex128 and complex64.

Edge cases the ring and the halo-indexed PRE_PSI rows must survive: grid-
aligned nodes (stencil width 2m+1), nodes at -1/2 and just below +1/2 (halo
wrap), batch counts around the ring's batch size, one dense cell (several
subproblems of one tile), and a single node.
"""

import numpy as np
import pytest

import paper_1810_09891_b200 as nf

pytestmark = pytest.mark.gpu

TOL = {"double": 1e-12, "single": 1e-5}


def e2(ref, got):
    ref = np.asarray(ref).astype(np.complex128).ravel()
    got = np.asarray(got).astype(np.complex128).ravel()
    return float(np.linalg.norm(ref - got) / np.linalg.norm(ref))


def nodes(d, n, M, seed, kind="uniform"):
    rng = np.random.default_rng(seed)
    if kind == "dense":  # everything in one cell of one tile
        return (rng.random((M, d)) * 0.9 / n[0] + 0.1 / n[0]).astype(np.float64)
    x = rng.random((M, d)) - 0.5
    if kind == "edges":
        k = max(1, M // 8)
        x[:k] = rng.integers(-n[0] // 2, n[0] // 2, size=(k, d)) / np.array(n)  # aligned
        x[k:2 * k, 0] = -0.5
        x[2 * k:3 * k, -1] = np.nextafter(0.5, 0.0)
    return x


def plan(N, n, m, x, precision, monkeypatch, tile=None):
    if tile:
        monkeypatch.setenv("NFFTK_TILE", str(tile))
    else:
        monkeypatch.delenv("NFFTK_TILE", raising=False)
    p = nf.Plan(N, x.shape[0], n=n, m=m, precision=precision)
    p.x = x
    p.precompute()
    return p


def check(p, N, n, m, x, oracle, precision):
    rng = np.random.default_rng(7)
    fh = rng.standard_normal(int(np.prod(N))) + 1j * rng.standard_normal(int(np.prod(N)))
    fs = rng.standard_normal(x.shape[0]) + 1j * rng.standard_normal(x.shape[0])
    assert p.mode == nf.MODE_TENSOR
    assert e2(oracle.trafo(N, n, m, x, fh), p.trafo(fh)) < TOL[precision]
    assert e2(oracle.adjoint(N, n, m, x, fs), p.adjoint(fs)) < TOL[precision]


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6])
def test_pipe_d3_every_cutoff(m, precision, oracle, monkeypatch):
    N, n = (8, 8, 8), (16, 16, 16)
    x = nodes(3, n, 3000, seed=m, kind="edges")
    p = plan(N, n, m, x, precision, monkeypatch, tile=8)
    assert p.tile == (8, 8, 8)
    check(p, N, n, m, x, oracle, precision)


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("m", [1, 2, 4, 6, 8])
def test_pipe_d2_every_cutoff(m, precision, oracle, monkeypatch):
    N, n = (16, 16), (32, 32)
    x = nodes(2, n, 3000, seed=10 + m, kind="edges")
    p = plan(N, n, m, x, precision, monkeypatch)
    assert p.tile == (32 - (2 * m + 1), 8)
    check(p, N, n, m, x, oracle, precision)


@pytest.mark.parametrize("M", [1, 15, 16, 17, 31, 32, 33, 64, 65])
def test_pipe_batch_boundaries(M, oracle, monkeypatch):
    N, n, m = (8, 8, 8), (16, 16, 16), 3
    x = nodes(3, n, M, seed=M)
    p = plan(N, n, m, x, "double", monkeypatch, tile=8)
    check(p, N, n, m, x, oracle, "double")
    N2, n2 = (16, 16), (32, 32)
    x2 = nodes(2, n2, M, seed=100 + M)
    p2 = plan(N2, n2, m, x2, "double", monkeypatch)
    assert p2.tile == (32 - (2 * m + 1), 8)
    check(p2, N2, n2, m, x2, oracle, "double")


@pytest.mark.parametrize("d", [2, 3])
def test_pipe_dense_cell_many_subproblems(d, oracle, monkeypatch):
    """5000 nodes in one cell: one tile split into several <= 1024-node
    subproblems, each flushing its own halo."""
    N, n, m = ((8, 8, 8), (16, 16, 16), 4) if d == 3 else ((16, 16), (32, 32), 6)
    x = nodes(d, n, 5000, seed=3, kind="dense")
    p = plan(N, n, m, x, "double", monkeypatch, tile=8 if d == 3 else None)
    check(p, N, n, m, x, oracle, "double")


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("d,m", [(3, 4), (3, 5), (3, 6), (2, 4), (2, 6)])
def test_dense_flush_matches_padded_fold(d, m, precision, oracle, monkeypatch):
    """The pipelined spreads reduce straight into the dense grid (rows
    wrapped periodically; c64 only for even m) -- same adjoint as the
    ghost-padded grid + fold path (NFFTK_NO_DENSE_FLUSH) and as the oracle,
    with nodes on every periodic boundary."""
    N, n = ((16, 16, 16), (32, 32, 32)) if d == 3 else ((32, 32), (64, 64))
    x = nodes(d, n, 4000, seed=20 + m, kind="edges")
    rng = np.random.default_rng(5)
    fs = rng.standard_normal(x.shape[0]) + 1j * rng.standard_normal(x.shape[0])
    dense = plan(N, n, m, x, precision, monkeypatch, tile=8 if d == 3 else None)
    monkeypatch.setenv("NFFTK_NO_DENSE_FLUSH", "1")
    padded = plan(N, n, m, x, precision, monkeypatch, tile=8 if d == 3 else None)
    monkeypatch.delenv("NFFTK_NO_DENSE_FLUSH")
    a, b = dense.adjoint(fs), padded.adjoint(fs)
    assert e2(b, a) < (1e-14 if precision == "double" else 1e-6)
    assert e2(oracle.adjoint(N, n, m, x, fs), a) < TOL[precision]


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("m,M,kind", [(6, 4000, "edges"), (4, 17, "uniform"), (8, 5000, "dense")])
def test_d2_sample_gather_matches_sorted_copy(m, M, kind, precision, oracle, monkeypatch):
    """k_spread2_pipe fetches its samples through perm itself (one cp.async per
    lane arriving on the batch's mbarrier); NFFTK_NO_GATHER reads the sorted
    copy k_permute_samples makes.  Same adjoint, also on replays."""
    N, n = (32, 32), (64, 64)
    x = nodes(2, n, M, seed=40 + m, kind=kind)
    rng = np.random.default_rng(6)
    fs = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    monkeypatch.delenv("NFFTK_NO_GATHER", raising=False)
    p = plan(N, n, m, x, precision, monkeypatch)
    a = [p.adjoint(fs) for _ in range(3)]
    monkeypatch.setenv("NFFTK_NO_GATHER", "1")
    b = p.adjoint(fs)
    monkeypatch.delenv("NFFTK_NO_GATHER")
    assert e2(oracle.adjoint(N, n, m, x, fs), a[0]) < TOL[precision]
    for v in a:
        assert e2(b, v) < (1e-14 if precision == "double" else 1e-6)


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("warps", ["1", "2"])
def test_d2_spread_warps_per_tile(warps, precision, oracle, monkeypatch):
    """k_spread2_pipe with one or two warps per tile (the second takes every
    other node of a batch; the register halos are added in the staging rows
    before the flush): same adjoint, nodes on the periodic boundaries and in
    one dense cell (several subproblems per tile)."""
    monkeypatch.setenv("NFFTK_SPREAD2_WARPS", warps)
    N, n, m = (32, 32), (64, 64), 6
    for kind, M in (("edges", 5000), ("dense", 3000), ("uniform", 1)):
        x = nodes(2, n, M, seed=50, kind=kind)
        p = plan(N, n, m, x, precision, monkeypatch)
        rng = np.random.default_rng(8)
        fs = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        ref = oracle.adjoint(N, n, m, x, fs)
        for _ in range(2):
            assert e2(ref, p.adjoint(fs)) < TOL[precision]
