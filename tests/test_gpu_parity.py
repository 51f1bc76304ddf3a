"""GPU parity tests: the CUDA path (through the C-ABI library) against the
CPU oracle (oracle/, pinned to the live reference) and the committed golden
vectors of the reference itself.

Tolerances (BASELINE.json north_star): relative l2 <= 1e-12 for complex128,
<= 1e-5 for complex64 (the reference has no complex64 path; its complex128
output is the oracle).  NDFT bands are m-aware.
"""

import ctypes
import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_1810_09891_b200 as nf
from paper_1810_09891_b200 import _lib
from paper_1810_09891_b200 import workloads as wl

pytestmark = pytest.mark.gpu

TOL128 = 1e-12
TOL64 = 1e-5

SMALL = np.load(os.path.join(GOLDEN, "small_cases.npz"))
NAMES = sorted({k.split("__")[0] for k in SMALL.files})


def case(name):
    return {f: SMALL[f"{name}__{f}"] for f in
            ("N", "n", "m", "x", "fhat", "f", "trafo", "adjoint", "order", "f1", "window",
             "ndft", "ndft_adjoint")}


def e2(ref, got):
    ref = np.asarray(ref).astype(np.complex128).ravel()
    got = np.asarray(got).astype(np.complex128).ravel()
    return float(np.linalg.norm(ref - got) / np.linalg.norm(ref))


def make_plan(c, precision="double", psi=None):
    p = nf.Plan(tuple(c["N"]), c["x"].shape[0], n=tuple(c["n"]), m=int(c["m"]),
                f1=int(c["f1"]), window=str(c["window"]), precision=precision)
    if psi is not None:
        p.set_psi_policy(psi)
    p.x = c["x"]
    p.precompute()
    return p


@pytest.fixture(scope="module")
def torch():
    import torch as t

    assert t.cuda.is_available(), "GPU tests need a CUDA device"
    return t


# ------------------------------------------------------------ golden cases
@pytest.mark.parametrize("name", NAMES)
def test_small_cases_vs_reference_goldens(name):
    c = case(name)
    p = make_plan(c)
    assert e2(c["trafo"], p.trafo(c["fhat"])) < TOL128
    assert e2(c["adjoint"], p.adjoint(c["f"])) < TOL128


@pytest.mark.parametrize("name", NAMES)
def test_small_cases_vs_oracle(name, oracle):
    c = case(name)
    lut = bool(int(c["f1"]) & nf.PRE_LIN_PSI) and not (int(c["f1"]) & (nf.PRE_PSI | nf.PRE_FULL_PSI))
    p = make_plan(c)
    ref_f = oracle.trafo(c["N"], c["n"], int(c["m"]), c["x"], c["fhat"], window=str(c["window"]), lut=lut)
    ref_a = oracle.adjoint(c["N"], c["n"], int(c["m"]), c["x"], c["f"], window=str(c["window"]), lut=lut)
    assert e2(ref_f, p.trafo(c["fhat"])) < TOL128
    assert e2(ref_a, p.adjoint(c["f"])) < TOL128


@pytest.mark.parametrize("name", [n for n in NAMES if int(case(n)["m"]) >= 6 and "lut" not in n])
def test_small_cases_vs_ndft(name):
    """Exact-sum check: the fast transform is within its own truncation error
    of the NDFT (reference E2 for the same inputs, 10x band)."""
    c = case(name)
    p = make_plan(c)
    band_f = max(10 * e2(c["ndft"], c["trafo"]), 1e-14)
    band_a = max(10 * e2(c["ndft_adjoint"], c["adjoint"]), 1e-14)
    assert e2(c["ndft"], p.trafo(c["fhat"])) < band_f
    assert e2(c["ndft_adjoint"], p.adjoint(c["f"])) < band_a


def test_table4_accuracy_d1_m8():
    """SPEC acceptance: E2 vs NDFT <= 1e-13 at m = 8 (Table 4 style)."""
    c = case("d1_m8")
    p = make_plan(c)
    assert e2(c["ndft"], p.trafo(c["fhat"])) < 1e-13
    assert e2(c["ndft_adjoint"], p.adjoint(c["f"])) < 1e-13


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_config_goldens_full(cfg):
    w = wl.CONFIGS[cfg]
    g = np.load(os.path.join(GOLDEN, f"{cfg}.npz"))
    p = nf.Plan(w.N, w.M, n=w.n, m=w.m)
    p.x = wl.nodes(w)
    p.precompute()
    assert e2(g["trafo"], p.trafo(wl.fhat(w))) < TOL128
    assert e2(g["adjoint"], p.adjoint(wl.samples(w))) < TOL128


def test_config_c3_golden_and_oracle(oracle):
    w = wl.CONFIGS["C3"]
    g = np.load(os.path.join(GOLDEN, "C3.npz"))
    x, fh, fs = wl.nodes(w), wl.fhat(w), wl.samples(w)
    p = nf.Plan(w.N, w.M, n=w.n, m=w.m)
    p.x = x
    p.precompute()
    f = p.trafo(fh)
    a = p.adjoint(fs)
    assert e2(g["trafo_sub"], f[g["trafo_idx"]]) < TOL128
    assert e2(g["adjoint_sub"], a[g["adjoint_idx"]]) < TOL128
    assert e2(oracle.trafo(w.N, w.n, w.m, x, fh), f) < TOL128
    assert e2(oracle.adjoint(w.N, w.n, w.m, x, fs), a) < TOL128


# ------------------------------------------------------------ complex64
@pytest.mark.parametrize("name", ["d1_m8", "d2_m8", "d2_clustered", "d3_m6", "d3_aligned", "d2_gauss"])
def test_complex64_vs_c128_reference(name):
    c = case(name)
    p = make_plan(c, precision="single")
    assert e2(c["trafo"], p.trafo(c["fhat"])) < TOL64
    assert e2(c["adjoint"], p.adjoint(c["f"])) < TOL64


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_complex64_configs(cfg, oracle):
    w = wl.CONFIGS[cfg]
    x, fh, fs = wl.nodes(w), wl.fhat(w), wl.samples(w)
    p = nf.Plan(w.N, w.M, n=w.n, m=w.m, precision="single")
    p.x = x
    p.precompute()
    assert e2(oracle.trafo(w.N, w.n, w.m, x, fh), p.trafo(fh)) < TOL64
    assert e2(oracle.adjoint(w.N, w.n, w.m, x, fs), p.adjoint(fs)) < TOL64


# ------------------------------------------------- modes / paths agree
def test_direct_and_tensor_modes_agree():
    """kernels.py modes DIRECT and TENSOR use identical factors (SPEC: <= 1e-14).

    The factors are bitwise identical; the sums are not: the TENSOR gather on
    the pipelined geometry walks stencil rows in a bank-conflict-free order
    (gridding.cu RowSched), the DIRECT batch kernel in natural order."""
    c = case("d3_m6")
    a = make_plan(c, psi=nf.MODE_DIRECT)
    b = make_plan(c, psi=nf.MODE_TENSOR)
    assert a.mode == nf.MODE_DIRECT and b.mode == nf.MODE_TENSOR
    assert e2(a.trafo(c["fhat"]), b.trafo(c["fhat"])) < 1e-14
    assert e2(a.adjoint(c["f"]), b.adjoint(c["f"])) < 1e-14


def test_full_psi_flag_maps_to_tensor():
    c = dict(case("d2_small"))
    c["f1"] = np.array(nf.PRE_PHI_HUT | nf.PRE_FULL_PSI)
    p = make_plan(c)
    assert p.mode == nf.MODE_TENSOR
    assert e2(c["trafo"], p.trafo(c["fhat"])) < TOL128


def test_lut_mode_tolerance_vs_exact():
    """PRE_LIN_PSI stays within the documented 1e-6 of the exact window (SPEC)."""
    c = case("d3_lut")
    exact = dict(c)
    exact["f1"] = np.array(nf.PRE_PHI_HUT | nf.PRE_PSI)
    assert e2(make_plan(exact).trafo(c["fhat"]), make_plan(c).trafo(c["fhat"])) < 1e-6


def test_device_path_equals_host_path(torch):
    c = case("d2_m8")
    p = make_plan(c)
    fh_host = p.trafo(c["fhat"])
    fh_dev = p.trafo(torch.from_numpy(c["fhat"]).cuda()).cpu().numpy()
    assert np.array_equal(fh_host, fh_dev)
    q = nf.Plan(tuple(c["N"]), c["x"].shape[0], n=tuple(c["n"]), m=int(c["m"]))
    q.x = torch.from_numpy(c["x"]).cuda()
    q.precompute()
    assert np.array_equal(q.trafo(c["fhat"]), fh_host)


@pytest.mark.parametrize("name", ["d3_m6", "d2_m8", "d1_m8"])
def test_cuda_graph_replay_matches_reference(name, torch):
    """trafo + adjoint captured once into a CUDA graph (as bench.py times the
    step) and replayed on new inputs copied into the captured buffers: the
    replay matches the reference goldens (ticket counters reset themselves)."""
    c = case(name)
    dev = torch.device("cuda", 0)
    p = make_plan(c)
    fh = torch.zeros(int(np.prod(c["N"])), dtype=torch.complex128, device=dev)
    fs = torch.zeros(c["x"].shape[0], dtype=torch.complex128, device=dev)
    f_out = torch.empty_like(fs)
    a_out = torch.empty_like(fh)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        p.trafo(fh, out=f_out)
        p.adjoint(fs, out=a_out)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        p.trafo(fh, out=f_out)
        p.adjoint(fs, out=a_out)
    for _ in range(2):
        fh.copy_(torch.from_numpy(c["fhat"].ravel()))
        fs.copy_(torch.from_numpy(c["f"].ravel()))
        g.replay()
        torch.cuda.synchronize()
        assert e2(c["trafo"], f_out.cpu().numpy()) < TOL128
        assert e2(c["adjoint"], a_out.cpu().numpy()) < TOL128


def test_cuda_graph_replay_c3_equals_eager(torch):
    """At the headline workload (persistent gridding kernels with dynamic
    subproblem tickets): graph replays give the eager trafo bit for bit and
    the eager adjoint to rounding (fp64 reductions in flush order)."""
    w = wl.CONFIGS["C3"]
    dev = torch.device("cuda", 0)
    p = nf.Plan(w.N, w.M, n=w.n, m=w.m)
    p.x = torch.from_numpy(wl.nodes(w)).to(dev)
    p.precompute()
    fh = torch.from_numpy(wl.fhat(w)).to(dev)
    fs = torch.from_numpy(wl.samples(w)).to(dev)
    f_ref = p.trafo(fh).clone()
    a_ref = p.adjoint(fs).clone()
    f_out = torch.empty_like(f_ref)
    a_out = torch.empty_like(a_ref)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        p.trafo(fh, out=f_out)
        p.adjoint(fs, out=a_out)
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(f_out, f_ref)
        assert e2(a_ref.cpu().numpy(), a_out.cpu().numpy()) < 1e-14


def test_trafo_deterministic_adjoint_stable():
    c = case("d3_m6")
    p = make_plan(c)
    assert np.array_equal(p.trafo(c["fhat"]), p.trafo(c["fhat"]))
    assert e2(p.adjoint(c["f"]), p.adjoint(c["f"])) < 1e-15


# -------------------------------------------------------------- C-ABI
def test_abi_spec_example():
    """SPEC cabi example: N=(4), M=1, x=0, f_hat_0 = 1 -> f = 1 within 1e-13."""
    lib = _lib.load()
    h = lib.nfftk_create(_lib.i32_array([4]), 1, 1)
    assert h > 0
    x = np.array([0.0])
    assert lib.nfftk_set_x(h, x.ctypes.data, 1) == 0, lib.nfftk_last_error_message(h)
    fh = np.array([0, 0, 0, 0, 1, 0, 0, 0], dtype=np.float64)
    assert lib.nfftk_set_fhat(h, fh.ctypes.data, 8) == 0
    assert lib.nfftk_trafo(h) == 0
    f = np.ctypeslib.as_array(ctypes.cast(lib.nfftk_get_f(h), ctypes.POINTER(ctypes.c_double)), (2,))
    assert abs(f[0] - 1.0) < 1e-13 and abs(f[1]) < 1e-13
    assert lib.nfftk_destroy(h) == 0


def test_abi_matches_python_api_bitwise():
    c = case("d3_m6")
    lib = _lib.load()
    d = int(c["x"].shape[1])
    h = lib.nfftk_create_advanced(_lib.i32_array(c["N"]), d, c["x"].shape[0],
                                  _lib.i32_array(c["n"]), int(c["m"]), int(c["f1"]), 0x41)
    assert h > 0
    x = np.ascontiguousarray(c["x"])
    assert lib.nfftk_set_x(h, x.ctypes.data, x.size) == 0
    fh = np.ascontiguousarray(c["fhat"]).view(np.float64)
    assert lib.nfftk_set_fhat(h, fh.ctypes.data, fh.size) == 0
    assert lib.nfftk_trafo(h) == 0
    M = x.shape[0]
    f = np.ctypeslib.as_array(ctypes.cast(lib.nfftk_get_f(h), ctypes.POINTER(ctypes.c_double)),
                              (2 * M,)).view(np.complex128)
    p = make_plan(c)
    assert np.array_equal(f, p.trafo(c["fhat"]))
    fs = np.ascontiguousarray(c["f"]).view(np.float64)
    assert lib.nfftk_set_f(h, fs.ctypes.data, fs.size) == 0
    assert lib.nfftk_adjoint(h) == 0
    K = int(np.prod(c["N"]))
    a = np.ctypeslib.as_array(ctypes.cast(lib.nfftk_get_fhat(h), ctypes.POINTER(ctypes.c_double)),
                              (2 * K,)).view(np.complex128)
    assert e2(c["adjoint"], a) < TOL128
    assert lib.nfftk_destroy(h) == 0


def test_abi_uploaded_buffers_and_chained_transforms(oracle):
    """nfftk_set_fhat / nfftk_set_f upload the library buffer while filling it
    and the following transform skips its host-to-device copy; a transform's
    result also stays on the device as the next one's input.  Every order of
    set / transform calls must see the latest buffer contents: repeated sets,
    transforms without a set in between (adjoint of the trafo result, trafo
    of the adjoint result), and replays of each captured graph."""
    N, n, m, M = (32, 32, 32), (64, 64, 64), 4, 150000
    rng = np.random.default_rng(21)
    x = rng.random((M, 3)) - 0.5
    K = int(np.prod(N))
    lib = _lib.load()
    h = lib.nfftk_create_advanced(_lib.i32_array(N), 3, M, _lib.i32_array(n), m, 0x1fd1, 0x41)
    assert h > 0
    assert lib.nfftk_set_x(h, x.ctypes.data, x.size) == 0, lib.nfftk_last_error_message(h)

    def cplx(k):
        return rng.standard_normal(k) + 1j * rng.standard_normal(k)

    def get(fn, k):
        return np.ctypeslib.as_array(ctypes.cast(fn(h), ctypes.POINTER(ctypes.c_double)),
                                     (2 * k,)).view(np.complex128).copy()

    for rep in range(3):
        fh_old, fh = cplx(K), cplx(K)
        for v in (fh_old, fh):  # the second set wins
            a = np.ascontiguousarray(v).view(np.float64)
            assert lib.nfftk_set_fhat(h, a.ctypes.data, a.size) == 0
        assert lib.nfftk_trafo(h) == 0
        f1 = get(lib.nfftk_get_f, M)
        assert e2(oracle.trafo(N, n, m, x, fh), f1) < TOL128
        assert np.array_equal(get(lib.nfftk_get_fhat, K), fh)
        # adjoint of the samples the trafo just produced (no set_f in between)
        assert lib.nfftk_adjoint(h) == 0
        a1 = get(lib.nfftk_get_fhat, K)
        assert e2(oracle.adjoint(N, n, m, x, f1), a1) < TOL128
        # trafo of the coefficients the adjoint just produced
        assert lib.nfftk_trafo(h) == 0
        assert e2(oracle.trafo(N, n, m, x, a1), get(lib.nfftk_get_f, M)) < TOL128
        # a fresh set_f replaces the chained samples
        fs = cplx(M)
        b = np.ascontiguousarray(fs).view(np.float64)
        assert lib.nfftk_set_f(h, b.ctypes.data, b.size) == 0
        assert lib.nfftk_adjoint(h) == 0
        assert e2(oracle.adjoint(N, n, m, x, fs), get(lib.nfftk_get_fhat, K)) < TOL128
    assert lib.nfftk_destroy(h) == 0


def test_abi_host_graph_replays_and_invalidation(oracle):
    """C-ABI calls on >= 1 MiB (pinned, library-owned) buffers run through a
    per-plan CUDA graph from the second call on: repeated calls reproduce the
    first, new nodes (set_x) invalidate the graph, results match the oracle."""
    N, n, m, M = (256, 256), (512, 512), 8, 65536
    rng = np.random.default_rng(5)
    lib = _lib.load()
    h = lib.nfftk_create_advanced(_lib.i32_array(N), 2, M, _lib.i32_array(n), m, 0x1fd1, 0x41)
    assert h > 0
    K = N[0] * N[1]
    fhc = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    fsc = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    fview = np.ctypeslib.as_array(ctypes.cast(lib.nfftk_get_f(h), ctypes.POINTER(ctypes.c_double)),
                                  (2 * M,)).view(np.complex128)
    aview = np.ctypeslib.as_array(ctypes.cast(lib.nfftk_get_fhat(h), ctypes.POINTER(ctypes.c_double)),
                                  (2 * K,)).view(np.complex128)
    for seed in (11, 12):
        x = np.ascontiguousarray(np.random.default_rng(seed).random((M, 2)) - 0.5)
        assert lib.nfftk_set_x(h, x.ctypes.data, x.size) == 0
        outs, adjs = [], []
        for _ in range(3):
            fh = np.ascontiguousarray(fhc).view(np.float64)
            assert lib.nfftk_set_fhat(h, fh.ctypes.data, fh.size) == 0
            assert lib.nfftk_trafo(h) == 0
            outs.append(fview.copy())
            fs = np.ascontiguousarray(fsc).view(np.float64)
            assert lib.nfftk_set_f(h, fs.ctypes.data, fs.size) == 0
            assert lib.nfftk_adjoint(h) == 0
            adjs.append(aview.copy())
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
        assert e2(adjs[0], adjs[2]) < 1e-14
        assert e2(oracle.trafo(N, n, m, x, fhc), outs[2]) < TOL128
        assert e2(oracle.adjoint(N, n, m, x, fsc), adjs[2]) < TOL128
    assert lib.nfftk_destroy(h) == 0


def test_abi_rank4_quirks():
    """Reference quirks: rank-4 set_x succeeds, trafo -> -2;
    rank-4 with PRE_FULL_PSI -> set_x -9."""
    lib = _lib.load()
    N = _lib.i32_array([4, 4, 4, 4])
    n = _lib.i32_array([8, 8, 8, 8])
    x = np.zeros(8)
    h = lib.nfftk_create_advanced(N, 4, 2, n, 2, 0x1fd1, 0x41)
    assert lib.nfftk_set_x(h, x.ctypes.data, 8) == 0
    assert lib.nfftk_trafo(h) == -2
    assert lib.nfftk_last_error_message(h) == b"fast transforms support d <= 3, got d=4"
    lib.nfftk_destroy(h)
    h = lib.nfftk_create_advanced(N, 4, 2, n, 2, 0x1fd1 | nf.PRE_FULL_PSI, 0x41)
    assert lib.nfftk_set_x(h, x.ctypes.data, 8) == -9
    lib.nfftk_destroy(h)


def test_state_errors():
    p = nf.Plan((16,), 4, n=(32,), m=4)
    with pytest.raises(nf.PlanStateError, match="no nodes"):
        p.trafo(np.zeros(16))
    p.set_nodes(np.zeros((4, 1)))
    with pytest.raises(nf.PlanStateError, match="not precomputed"):
        p.trafo(np.zeros(16))
    p.precompute()
    with pytest.raises(nf.ShapeError):
        p.trafo(np.zeros(15))
    assert p.trafo(np.zeros((4, 4))).shape == (4,)


# -------------------------------------------------------- properties
@pytest.mark.parametrize("d", [1, 2, 3])
def test_adjoint_identity(d):
    """SPEC: |<A fh, f> - <fh, A^H f>| / (|fh| |f|) <= 1e-12 over random instances."""
    rng = np.random.default_rng(100 + d)
    for _ in range(10):
        N = tuple(int(v) for v in 2 * rng.integers(2, 9, d))
        n = tuple(2 * v for v in N)
        m = int(rng.integers(1, min(n) // 2))
        m = max(1, min(m, (min(n) - 1) // 2, 8))
        M = int(rng.integers(1, 300))
        p = nf.Plan(N, M, n=n, m=m)
        p.x = rng.random((M, d)) - 0.5
        p.precompute()
        K = int(np.prod(N))
        fh = rng.standard_normal(K) + 1j * rng.standard_normal(K)
        f = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        lhs = np.vdot(f, p.trafo(fh))
        rhs = np.vdot(p.adjoint(f), fh)
        assert abs(lhs - rhs) / (np.linalg.norm(fh) * np.linalg.norm(f)) < 1e-12


def test_node_order_matches_lexsort(oracle):
    for name in ("d2_aligned", "d3_aniso", "d2_clustered"):
        c = case(name)
        p = make_plan(c)
        assert np.array_equal(p.node_order, c["order"])
        # the tables precompute returns (plan.py:296) carry the same order,
        # materialised on first access
        assert np.array_equal(p.precompute().node_order, c["order"])


def test_window_eval_counter():
    c = dict(case("d2_aligned"))
    c["f1"] = np.array(nf.PRE_PHI_HUT)  # DIRECT mode: counts evaluations
    p = make_plan(c)
    p.trafo(c["fhat"])
    lo, width = nf.indexing.node_ranges(c["x"], tuple(c["n"]), int(c["m"]))
    assert p.window_evals_last == int(width.sum())
    p.adjoint(c["f"])
    assert p.window_evals_total == 2 * int(width.sum())
    assert p.window_evals_total <= 2 * (2 * int(c["m"]) + 1) ** 2 * c["x"].shape[0] * 2


def test_tiny_grid_halo_wraps(oracle):
    """Halo larger than the grid (T + 2m + 1 > n): cells alias onto themselves."""
    rng = np.random.default_rng(3)
    for N, n, m in [((4,), (8,), 3), ((4, 4), (8, 10), 3), ((2, 2, 2), (8, 8, 8), 3)]:
        M = 57
        x = rng.random((M, len(N))) - 0.5
        x[0] = -0.5
        K = int(np.prod(N))
        fh = rng.standard_normal(K) + 1j * rng.standard_normal(K)
        fs = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        p = nf.Plan(N, M, n=n, m=m)
        p.x = x
        p.precompute()
        assert e2(oracle.trafo(N, n, m, x, fh), p.trafo(fh)) < TOL128
        assert e2(oracle.adjoint(N, n, m, x, fs), p.adjoint(fs)) < TOL128


def test_dense_single_cell_nodes(oracle):
    """Many nodes in one cell (heavy subproblem splitting + contention)."""
    rng = np.random.default_rng(4)
    N, n, m, M = (32, 32), (64, 64), 6, 5000
    x = 0.01 + 1e-4 * rng.random((M, 2))
    fh = rng.standard_normal(1024) + 1j * rng.standard_normal(1024)
    fs = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    p = nf.Plan(N, M, n=n, m=m)
    p.x = x
    p.precompute()
    assert e2(oracle.trafo(N, n, m, x, fh), p.trafo(fh)) < TOL128
    assert e2(oracle.adjoint(N, n, m, x, fs), p.adjoint(fs)) < TOL128


# ------------------------------------------------- full-size properties
@pytest.mark.parametrize("cfg", ["C4", "C5"])
def test_full_size_trafo_subsample_and_adjoint_identity(cfg, oracle, torch):
    """At BASELINE sizes: trafo on a node subsample equals the oracle run on
    those nodes (trafo is per-node independent), and the adjoint satisfies
    the adjoint identity against the trafo at full size."""
    w = wl.CONFIGS[cfg]
    x = wl.nodes(w)
    fh = wl.fhat(w)
    p = nf.Plan(w.N, w.M, n=w.n, m=w.m)
    p.x = torch.from_numpy(x).cuda()
    p.precompute()
    fh_d = torch.from_numpy(fh).cuda()
    f = p.trafo(fh_d)
    idx = np.sort(np.random.default_rng(9).choice(w.M, 512, replace=False))
    ref = oracle.trafo(w.N, w.n, w.m, x[idx], fh)
    assert e2(ref, f[torch.from_numpy(idx).cuda()].cpu().numpy()) < TOL128
    g = torch.from_numpy(wl.samples(w)).cuda()
    a = p.adjoint(g)
    lhs = torch.vdot(g, f).item()
    rhs = torch.vdot(a, fh_d).item()
    scale = torch.linalg.norm(fh_d).item() * torch.linalg.norm(g).item()
    assert abs(lhs - rhs) / scale < 1e-12


def test_distributed_plan_single_rank_matches_plan(torch):
    """GPU engine of the node-sharded orchestration (world = 1): bound grid,
    spread, finish reproduce Plan.adjoint / trafo."""
    from paper_1810_09891_b200.distributed import DistributedPlan

    c = case("d3_m6")
    dev = torch.device("cuda", 0)
    dp = DistributedPlan(tuple(c["N"]), c["x"].shape[0], n=tuple(c["n"]), m=int(c["m"]), device=dev)
    dp.set_nodes(torch.from_numpy(c["x"]).to(dev))
    dp.precompute()
    f = dp.trafo(torch.from_numpy(c["fhat"]).to(dev)).cpu().numpy()
    a = dp.adjoint(torch.from_numpy(c["f"]).to(dev)).cpu().numpy()
    assert e2(c["trafo"], f) < TOL128
    assert e2(c["adjoint"], a) < TOL128
    dp.close()


# ------------------------------------------------ PrecomputeTables contents
@pytest.mark.parametrize("name", ["d1_small", "d2_aligned", "d3_aligned", "d3_m6"])
def test_tables_psi_in_reference_layout(name, oracle):
    """tables.psi (M, d, 2m+1) and the PRE_FULL_PSI tables (plan.py:109-121,
    kernels.py:56-119) materialised from the device in natural node order:
    the window at x - (lo + t)/n, zero past the width; products in
    lexicographic order with their flat wrapped cells."""
    c = dict(case(name))
    c["f1"] = np.array(nf.PRE_PHI_HUT | nf.PRE_PSI | nf.PRE_FULL_PSI)
    p = make_plan(c)
    t = p.tables
    x, n, m = c["x"], tuple(int(v) for v in c["n"]), int(c["m"])
    M, d = x.shape
    K = 2 * m + 1
    lo, width = oracle.node_ranges(n, m, x)
    b = [oracle.window_b(0, int(Ni), int(ni), m) for Ni, ni in zip(c["N"], n)]
    ref = np.zeros((M, d, K))
    for j in range(M):
        for i in range(d):
            for k in range(width[j, i]):
                ref[j, i, k] = oracle.window_factor(0, x[j, i] - (lo[j, i] + k) / n[i], n[i], m, b[i])
    assert t.psi.shape == (M, d, K)
    assert np.allclose(t.psi, ref, rtol=1e-14, atol=0)
    vals, idx, counts = t.psi_full_vals, t.psi_full_idx, t.psi_full_counts
    assert vals.shape == (M, K ** d) and idx.shape == (M, K ** d)
    assert np.array_equal(counts, np.prod(width, axis=1))
    for j in range(M):
        cells = [np.mod(lo[j, i] + np.arange(width[j, i]), n[i]) for i in range(d)]
        facs = [t.psi[j, i, :width[j, i]] for i in range(d)]
        prod, flat = facs[0], cells[0]
        for i in range(1, d):
            prod = (prod[:, None] * facs[i][None, :]).ravel()
            flat = (flat[:, None] * n[i] + cells[i][None, :]).ravel()
        assert np.array_equal(vals[j, :counts[j]], prod)
        assert np.array_equal(idx[j, :counts[j]], flat)
        assert not vals[j, counts[j]:].any() and not idx[j, counts[j]:].any()


def test_tables_lut_and_absent_entries(oracle):
    from paper_1810_09891_b200.plan import LUT_SIZE

    c = dict(case("d2_lut"))
    p = make_plan(c)
    t = p.tables
    assert t.psi is None and t.psi_full_vals is None
    n, m = tuple(int(v) for v in c["n"]), int(c["m"])
    assert t.lut.shape == (2, LUT_SIZE + 1)
    for i in range(2):
        b = oracle.window_b(0, int(c["N"][i]), n[i], m)
        h = (m / n[i]) / LUT_SIZE
        for s in (0, 1, 777, LUT_SIZE):
            ref = oracle.window_factor(0, s * h, n[i], m, b)
            assert abs(t.lut[i, s] - ref) <= 1e-15 * abs(ref)
        assert t.lut_steps[i] == LUT_SIZE / (m / n[i])
