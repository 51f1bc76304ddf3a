"""Parity of the residue-owned d=3 spread (residue.cu: k_spread_res,
k_wide_nodes; the interp of these plans is k_interp_pipe on the same node
order) against the CPU oracle: 8^3 tiles, every cutoff 1..6 in complex128 and
the even ones in complex64; most cases at m = 4 (the C5 geometry).  Cases: grids
whose tiles divide n and do not (partial last tiles), nodes on every periodic
boundary, grid-aligned nodes (2m+1 wide stencils: the k_wide_nodes pass), one
dense cell (several subproblems of one tile), clustered nodes, node counts
around the ring's batch sizes, every ring shape, and replays of one plan
(ticket counters, row state)."""

import numpy as np
import pytest

import paper_1810_09891_b200 as nf

pytestmark = pytest.mark.gpu

M4 = 4


def e2(ref, got):
    ref = np.asarray(ref).astype(np.complex128).ravel()
    got = np.asarray(got).astype(np.complex128).ravel()
    return float(np.linalg.norm(ref - got) / np.linalg.norm(ref))


def nodes(n, M, seed, kind="uniform"):
    rng = np.random.default_rng(seed)
    if kind == "dense":  # everything in one cell of one tile
        return rng.random((M, 3)) * 0.9 / n[0] + 0.1 / n[0]
    if kind == "clustered":
        c = rng.random((4, 3)) - 0.5
        x = c[rng.integers(0, 4, M)] + 0.03 * rng.standard_normal((M, 3))
        return (x + 0.5) % 1.0 - 0.5
    x = rng.random((M, 3)) - 0.5
    if kind == "edges":
        k = max(1, M // 8)
        x[:k] = rng.integers(-n[0] // 2, n[0] // 2, size=(k, 3)) / np.array(n)  # aligned: wide stencils
        x[k:2 * k, 0] = -0.5
        x[2 * k:3 * k, -1] = np.nextafter(0.5, 0.0)
        x[3 * k:4 * k, 1] = rng.integers(-n[1] // 2, n[1] // 2, size=k) / n[1]  # wide in one dim only
    return x


TOL = {"double": 1e-12, "single": 1e-5}


def plan(N, n, x, monkeypatch, variant=None, m=M4, precision="double"):
    monkeypatch.setenv("NFFTK_TILE", "8")
    monkeypatch.setenv("NFFTK_RES_ANY_M", "1")  # cutoffs other than 4 take the row kernels by default
    if variant is not None:
        monkeypatch.setenv("NFFTK_RES_VARIANT", str(variant))
    else:
        monkeypatch.delenv("NFFTK_RES_VARIANT", raising=False)
    p = nf.Plan(N, x.shape[0], n=n, m=m, precision=precision)
    p.x = x
    p.precompute()
    assert p.tile == (8, 8, 8) and p.gridding == "residue"
    return p


def check(p, N, n, x, oracle, reps=1, m=M4, precision="double"):
    rng = np.random.default_rng(7)
    fh = rng.standard_normal(int(np.prod(N))) + 1j * rng.standard_normal(int(np.prod(N)))
    fs = rng.standard_normal(x.shape[0]) + 1j * rng.standard_normal(x.shape[0])
    rt = oracle.trafo(N, n, m, x, fh)
    ra = oracle.adjoint(N, n, m, x, fs)
    for _ in range(reps):
        assert e2(rt, p.trafo(fh)) < TOL[precision]
        assert e2(ra, p.adjoint(fs)) < TOL[precision]


@pytest.mark.parametrize("m,precision", [(1, "double"), (2, "double"), (3, "double"), (4, "double"), (5, "double"),
                                         (6, "double"), (2, "single"), (4, "single"), (6, "single")])
@pytest.mark.parametrize("n1,kind", [(32, "edges"), (28, "uniform"), (40, "clustered")])
def test_residue_every_cutoff(m, precision, n1, kind, oracle, monkeypatch):
    """Every instantiated cutoff and precision: nodes on the periodic
    boundaries and grid-aligned (wide) nodes, a grid the tiles do not divide,
    clustered nodes (tiles split into several subproblems)."""
    N, n = (8, 8, 8), (n1, n1, n1)
    x = nodes(n, 12000, seed=3 * m + n1, kind=kind)
    p = plan(N, n, x, monkeypatch, m=m, precision=precision)
    check(p, N, n, x, oracle, m=m, precision=precision, reps=2)


def test_residue_odd_cutoff_single_uses_row_kernels(monkeypatch):
    """complex64 bulk reductions need 16-byte pieces: odd m (odd row start)
    stays on the row-per-thread kernels."""
    monkeypatch.setenv("NFFTK_TILE", "8")
    monkeypatch.setenv("NFFTK_RES_ANY_M", "1")
    x = nodes((32, 32, 32), 5000, seed=1)
    p = nf.Plan((8, 8, 8), 5000, n=(32, 32, 32), m=3, precision="single")
    p.x = x
    p.precompute()
    assert p.gridding == "pipe"


@pytest.mark.parametrize("n1", [24, 32, 20, 36, 18])
def test_residue_grids(n1, oracle, monkeypatch):
    """n a multiple of the tile edge, and not (the last tile of a dim is partial)."""
    N, n = (8, 8, 8), (n1, n1, n1)
    x = nodes(n, 6000, seed=n1, kind="edges")
    p = plan(N, n, x, monkeypatch)
    assert p.wide_nodes >= 6000 // 8
    check(p, N, n, x, oracle)


def test_residue_anisotropic(oracle, monkeypatch):
    N, n = (8, 16, 12), (24, 40, 32)
    x = nodes(n, 9000, seed=3)
    check(plan(N, n, x, monkeypatch), N, n, x, oracle)


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["uniform", "clustered", "dense"])
def test_residue_node_sets(kind, variant, oracle, monkeypatch):
    N, n = (16, 16, 16), (32, 32, 32)
    x = nodes(n, 20000 if kind != "dense" else 5000, seed=11, kind=kind)
    p = plan(N, n, x, monkeypatch, variant=variant)
    check(p, N, n, x, oracle, reps=2)


@pytest.mark.parametrize("M", [1, 3, 15, 16, 17, 31, 32, 33, 63, 64, 65, 97])
def test_residue_batch_boundaries(M, oracle, monkeypatch):
    N, n = (8, 8, 8), (24, 24, 24)
    x = nodes(n, M, seed=M)
    check(plan(N, n, x, monkeypatch), N, n, x, oracle)


def test_residue_all_nodes_aligned(oracle, monkeypatch):
    """Every stencil 2m+1 wide: the residue spread skips every node and
    k_wide_nodes does the whole adjoint."""
    N, n = (8, 8, 8), (24, 24, 24)
    rng = np.random.default_rng(5)
    x = rng.integers(-12, 12, size=(500, 3)) / 24.0
    p = plan(N, n, x, monkeypatch)
    assert p.wide_nodes == 500
    check(p, N, n, x, oracle)


def test_residue_matches_row_kernels(oracle, monkeypatch):
    """Same plan parameters through the row-per-thread pipelined kernels
    (NFFTK_NO_RES): the two B / B^H implementations agree to rounding."""
    N, n = (16, 16, 16), (32, 32, 32)
    x = nodes(n, 30000, seed=21, kind="edges")
    rng = np.random.default_rng(9)
    fh = rng.standard_normal(16 ** 3) + 1j * rng.standard_normal(16 ** 3)
    fs = rng.standard_normal(30000) + 1j * rng.standard_normal(30000)
    p = plan(N, n, x, monkeypatch)
    monkeypatch.setenv("NFFTK_NO_RES", "1")
    q = nf.Plan(N, 30000, n=n, m=M4)
    q.x = x
    q.precompute()
    monkeypatch.delenv("NFFTK_NO_RES")
    assert q.gridding == "pipe"
    assert e2(q.trafo(fh), p.trafo(fh)) < 1e-13
    assert e2(q.adjoint(fs), p.adjoint(fs)) < 1e-13


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("kind,M", [("edges", 30000), ("dense", 3000), ("uniform", 33)])
def test_residue_sample_gather_matches_sorted_copy(kind, M, precision, oracle, monkeypatch):
    """Warp 0 gathers each batch's samples from the caller's array, one
    cp.async per lane arriving on the batch's mbarrier (default);
    NFFTK_NO_GATHER reads them from the sorted copy k_permute_samples makes.
    Same FMA order per row: the adjoints agree to the rounding of the row
    reductions, also across replays and with wide (k_wide_nodes) nodes."""
    N, n = (16, 16, 16), (32, 32, 32)
    x = nodes(n, M, seed=31, kind=kind)
    rng = np.random.default_rng(13)
    fs = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    monkeypatch.delenv("NFFTK_NO_GATHER", raising=False)
    p = plan(N, n, x, monkeypatch, precision=precision)
    a = [p.adjoint(fs) for _ in range(3)]
    monkeypatch.setenv("NFFTK_NO_GATHER", "1")
    b = p.adjoint(fs)
    monkeypatch.delenv("NFFTK_NO_GATHER")
    assert e2(oracle.adjoint(N, n, M4, x, fs), a[0]) < TOL[precision]
    # the flushes are floating-point reductions whose order varies run to run
    for v in a:
        assert e2(b, v) < (1e-14 if precision == "double" else 1e-6)
