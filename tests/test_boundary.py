"""Drop-in boundary checks that need no GPU: the C-ABI library loads, exports
every symbol include/nfftk.h declares, and reproduces the reference's
handle / error-code semantics (cabi.py:39-245, abi.py:162-275) for every path
that does not launch a kernel.  Also the Python Plan's validation order and
exception classes (plan.py:138-186)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
import paper_1810_09891_b200 as nf
from paper_1810_09891_b200 import _lib

HEADER = os.path.join(ROOT, "include", "nfftk.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(nfftk_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 13
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_reference_symbols_present():
    ref = ["nfftk_abi_version", "nfftk_create", "nfftk_create_advanced", "nfftk_set_x",
           "nfftk_set_fhat", "nfftk_set_f", "nfftk_trafo", "nfftk_adjoint", "nfftk_get_f",
           "nfftk_get_fhat", "nfftk_last_error", "nfftk_last_error_message", "nfftk_destroy"]
    assert set(ref) <= set(header_symbols())


@pytest.fixture
def lib():
    return _lib.load()


def ivec(*v):
    return _lib.i32_array(v)


def test_abi_version(lib):
    assert lib.nfftk_abi_version() == b"0.1.0"


@pytest.mark.parametrize("args,code", [
    (((16,), 0, 10), -3),            # rank < 1 (abi.py:196-197)
    (((15,), 1, 10), -3),            # odd bandlimit -> InvalidBandlimitError
    (((16,), 1, 0), -9),             # M = 0 -> base NfftError -> internal (cabi quirk)
])
def test_create_codes(lib, args, code):
    N, rank, M = args
    assert lib.nfftk_create(ivec(*N), rank, M) == code


@pytest.mark.parametrize("n,m,f1,code", [
    ((16,), 4, 0xfd1, -3),           # n <= N  -> OversamplingError
    ((33,), 4, 0xfd1, -3),           # odd n   -> OversamplingError
    ((32,), 16, 0xfd1, -3),          # 2m+1 > n -> CutoffError
    ((32,), 0, 0xfd1, -3),           # m < 1   -> CutoffError
    ((32,), 4, 0x2, -3),             # FG_PSI  -> UnsupportedFlagError
    ((32,), 4, 1 << 20, -3),         # unknown bit
])
def test_create_advanced_codes(lib, n, m, f1, code):
    assert lib.nfftk_create_advanced(ivec(16), 1, 4, ivec(*n), m, f1, 0x41) == code


def test_handle_lifecycle_and_buffers(lib):
    h = lib.nfftk_create_advanced(ivec(4), 1, 1, ivec(16), 2, 0xfd1, 0x41)
    assert h > 0
    assert lib.nfftk_last_error(h) == 0
    f = lib.nfftk_get_f(h)
    fh = lib.nfftk_get_fhat(h)
    assert f and fh
    assert np.ctypeslib.as_array(ctypes.cast(f, ctypes.POINTER(ctypes.c_double)), (2,)).tolist() == [0, 0]
    vals = np.array([0, 0, 0, 0, 1, 0, 0, 0], dtype=np.float64)
    assert lib.nfftk_set_fhat(h, vals.ctypes.data, 8) == 0
    view = np.ctypeslib.as_array(ctypes.cast(lib.nfftk_get_fhat(h), ctypes.POINTER(ctypes.c_double)), (8,))
    assert view.tolist() == vals.tolist()
    # wrong length: -2, buffer unchanged (cabi.py:149-160)
    bad = np.ones(6)
    assert lib.nfftk_set_fhat(h, bad.ctypes.data, 6) == -2
    assert lib.nfftk_last_error(h) == -2
    assert lib.nfftk_last_error_message(h) == b"fhat needs 8 interleaved doubles, got 6"
    assert view.tolist() == vals.tolist()
    assert lib.nfftk_set_f(h, bad.ctypes.data, 6) == -2
    assert lib.nfftk_last_error_message(h) == b"f needs 2 interleaved doubles, got 6"
    # set_x shape / range errors happen before any device work
    x2 = np.zeros(2)
    assert lib.nfftk_set_x(h, x2.ctypes.data, 2) == -2
    assert lib.nfftk_last_error_message(h) == b"need 1 coordinates (1 nodes x 1), got 2"
    xb = np.array([0.5])
    assert lib.nfftk_set_x(h, xb.ctypes.data, 1) == -3
    assert lib.nfftk_last_error_message(h) == b"node 0 coordinate 0.5 outside [-1/2, 1/2)"
    # transforms before nodes: PlanStateError -> -3
    assert lib.nfftk_trafo(h) == -3
    assert lib.nfftk_last_error_message(h) == b"plan has no nodes; call set_nodes() first"
    assert lib.nfftk_adjoint(h) == -3
    # success resets the stored error
    assert lib.nfftk_set_fhat(h, vals.ctypes.data, 8) == 0
    assert lib.nfftk_last_error(h) == 0
    assert lib.nfftk_last_error_message(h) == b""
    assert lib.nfftk_destroy(h) == 0
    assert lib.nfftk_destroy(h) == -1
    assert not lib.nfftk_get_f(h)
    assert lib.nfftk_last_error(h) == -1
    assert lib.nfftk_last_error_message(h) == b"invalid handle"
    assert lib.nfftk_trafo(h) == -1


def test_rank4_plan_creates(lib):
    h = lib.nfftk_create(ivec(4, 4, 4, 4), 4, 3)
    assert h > 0
    assert lib.nfftk_destroy(h) == 0


def test_handle_stress_no_leak(lib):
    """cabi SPEC invariant: 10^4 create/use/destroy cycles leak nothing."""
    h0, b0 = lib.nfftk_live_handles(), lib.nfftk_live_buffers()
    vals = np.zeros(8)
    for _ in range(10_000):
        h = lib.nfftk_create_advanced(ivec(4), 1, 1, ivec(16), 2, 0xfd1, 0x41)
        assert h > 0
        assert lib.nfftk_set_fhat(h, vals.ctypes.data, 8) == 0
        assert lib.nfftk_destroy(h) == 0
    assert lib.nfftk_live_handles() == h0
    assert lib.nfftk_live_buffers() == b0


# ------------------------------------------------------------ Python Plan
@pytest.mark.parametrize("kwargs,exc,msg", [
    (dict(N=(16,), M=10, n=(16,)), nf.OversamplingError, "need n_i > N_i, got n=(16,) for N=(16,)"),
    (dict(N=(16,), M=10, n=(17,)), nf.OversamplingError, "FFT lengths must be even, got 17"),
    (dict(N=(15,), M=10), nf.InvalidBandlimitError, "bandlimit entries must be even and >= 2, got 15"),
    (dict(N=(), M=10), nf.InvalidBandlimitError, "bandlimit vector is empty"),
    (dict(N=(16,), M=0), nf.NfftError, "node count must be >= 1, got 0"),
    (dict(N=(16,), M=5, n=(32,), m=20), nf.CutoffError, "cutoff 20 needs 2m+1 <= min(n) = 32"),
    (dict(N=(16,), M=5, n=(32,), m=0), nf.CutoffError, "cutoff must be >= 1, got 0"),
    (dict(N=(16,), M=5, f1=2), nf.UnsupportedFlagError, None),
    (dict(N=(16,), M=5, f1=1 << 20), nf.InvalidFlagError, "unknown f1 bits: 0x100000"),
    (dict(N=(16,), M=5, f1=-1), nf.InvalidFlagError, None),
    (dict(N=(16, 16), M=5, n=(32,)), nf.ShapeError, "n has 1 dims, N has 2"),
    (dict(N=(16,), M=5, window="bspline"), nf.NfftError, None),
])
def test_plan_validation(kwargs, exc, msg):
    with pytest.raises(exc) as info:
        nf.Plan(**kwargs)
    if msg is not None:
        assert str(info.value) == msg


def test_unsupported_flag_is_invalid_flag():
    assert issubclass(nf.UnsupportedFlagError, nf.InvalidFlagError)


def test_plan_defaults():
    p = nf.Plan((16,), 5)
    assert p.n == (32,) and p.m == 8          # 2**(ceil(log2 16)+1) >= 2*8+2 (plan.py:144-155)
    assert p.f1 == 0xfd1 and p.f2 == 0x41
    q = nf.Plan((1024,), 5)
    assert q.n == (2048,) and q.m == 8
    r = nf.Plan((16, 16), 5, n=(20, 40))
    assert r.m == 8 and r.f1 == 0x1fd1        # m = min(8, (20-1)//2) = 9 -> 8
    s = nf.Plan((8,), 5, n=(10,))
    assert s.m == 4                            # (10-1)//2
    assert repr(q) == "Plan(N=(1024,), M=5, n=(2048,), m=8, f1=0xfd1, f2=0x41, window='kaiserbessel')"
    assert nf.default_f1(1) == 0xfd1 and nf.default_f1(3) == 0x1fd1
    assert nf.default_n((1000, 64, 6)) == (2048, 128, 16)


def test_plan_node_checks_without_gpu():
    p = nf.Plan((16, 16), 3)
    with pytest.raises(nf.ShapeError):
        p.x = np.zeros((3, 3))
    bad = np.zeros((3, 2))
    bad[1, 1] = -0.75
    with pytest.raises(nf.NodeRangeError) as info:
        p.x = bad
    assert str(info.value) == "node 1 coordinate -0.75 outside [-1/2, 1/2)"
    with pytest.raises(nf.PlanStateError):
        p.trafo(np.zeros(256))
    with pytest.raises(nf.PlanStateError):
        p.precompute()


def test_window_model_pins():
    pins = np.load(os.path.join(ROOT, "tests", "golden", "pins.npz"))
    for kind in ("kaiserbessel", "gaussian"):
        w = nf.WindowModel.make(kind, (64,), (128,), 6)
        key = f"{kind}_64_128_6"
        assert w.b[0] == pins["b_" + key][0]
        assert np.allclose(w.phi_hat_table(0, 32), pins["phihat_" + key], rtol=1e-15, atol=0)
        assert np.allclose(w.phi(pins["phi_t_" + key]), pins["phi_" + key], rtol=2e-15, atol=0)


def test_indexing_helpers():
    assert nf.index_set((4,)).ravel().tolist() == [-2, -1, 0, 1]
    assert [tuple(k) for k in nf.index_set((2, 2))] == [(-1, -1), (-1, 0), (0, -1), (0, 0)]
    assert nf.linear_index((0, 0), (2, 2)) == 3
    for i in range(24):
        assert nf.linear_index(nf.multi_index(i, (4, 6)), (4, 6)) == i
    x = np.array([[0.0]])
    assert nf.transposed_members((0,), x, (8,), 1).tolist() == [0]
    assert nf.transposed_members((-4,), x, (8,), 1).tolist() == []


def test_metrics():
    assert nf.error_e2([1, 0], [1, 0]) == 0.0
    assert nf.error_e2([3, 4], [0, 0]) == 1.0
    with pytest.raises(nf.UndefinedMetricError):
        nf.error_e2([0, 0], [1, 1])

    class P:
        m, d, M, num_freqs, grid_size = 8, 1, 1024, 512, 1024
    assert nf.cost_estimate(P) == 512 + 1024 * 10 + 2 * 17 * 1024
