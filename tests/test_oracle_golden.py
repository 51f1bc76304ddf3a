"""Pin the CPU oracle (oracle/) against golden vectors produced by the live
reference package (tests/golden/make_golden.py) and against the reference's
own test pins.  CPU only."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1810_09891_b200 import workloads as wl

SMALL = np.load(os.path.join(GOLDEN, "small_cases.npz"))
PINS = np.load(os.path.join(GOLDEN, "pins.npz"))
NAMES = sorted({k.split("__")[0] for k in SMALL.files})


def case(name):
    return {f: SMALL[f"{name}__{f}"] for f in
            ("N", "n", "m", "x", "fhat", "f", "trafo", "adjoint", "order", "f1", "window",
             "ndft", "ndft_adjoint")}


def lut_mode(c):
    f1 = int(c["f1"])
    return bool(f1 & 4) and not (f1 & 0x30)


@pytest.mark.parametrize("name", NAMES)
def test_oracle_trafo_matches_reference(oracle, name):
    c = case(name)
    out = oracle.trafo(c["N"], c["n"], int(c["m"]), c["x"], c["fhat"], window=str(c["window"]),
                       lut=lut_mode(c))
    assert oracle.error_e2(c["trafo"], out) < 1e-14


@pytest.mark.parametrize("name", NAMES)
def test_oracle_adjoint_matches_reference(oracle, name):
    c = case(name)
    out = oracle.adjoint(c["N"], c["n"], int(c["m"]), c["x"], c["f"], window=str(c["window"]),
                         lut=lut_mode(c))
    assert oracle.error_e2(c["adjoint"], out) < 1e-14


@pytest.mark.parametrize("name", NAMES)
def test_oracle_ndft_matches_reference(oracle, name):
    c = case(name)
    assert oracle.error_e2(c["ndft"], oracle.ndft(c["N"], c["x"], c["fhat"])) < 1e-13
    assert oracle.error_e2(c["ndft_adjoint"], oracle.ndft_adjoint(c["N"], c["x"], c["f"])) < 1e-13


@pytest.mark.parametrize("name", [n for n in NAMES if case(n)["order"].size])
def test_oracle_node_order_matches_lexsort(oracle, name):
    c = case(name)
    assert np.array_equal(oracle.node_order(c["n"], c["x"]), c["order"])


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_oracle_config_goldens(oracle, cfg):
    w = wl.CONFIGS[cfg]
    g = np.load(os.path.join(GOLDEN, f"{cfg}.npz"))
    x = wl.nodes(w)
    assert oracle.error_e2(g["trafo"], oracle.trafo(w.N, w.n, w.m, x, wl.fhat(w))) < 1e-14
    assert oracle.error_e2(g["adjoint"], oracle.adjoint(w.N, w.n, w.m, x, wl.samples(w))) < 1e-14


def test_oracle_c3_golden_subsample(oracle):
    w = wl.CONFIGS["C3"]
    g = np.load(os.path.join(GOLDEN, "C3.npz"))
    x = wl.nodes(w)
    f = oracle.trafo(w.N, w.n, w.m, x, wl.fhat(w))
    a = oracle.adjoint(w.N, w.n, w.m, x, wl.samples(w))
    assert oracle.error_e2(g["trafo_sub"], f[g["trafo_idx"]]) < 1e-14
    assert oracle.error_e2(g["adjoint_sub"], a[g["adjoint_idx"]]) < 1e-14
    assert abs(np.linalg.norm(f) - g["norm_f"]) / g["norm_f"] < 1e-14
    assert abs(np.linalg.norm(a) - g["norm_fhat"]) / g["norm_fhat"] < 1e-14


def test_oracle_accuracy_vs_ndft_m8(oracle):
    """Table-4 style accuracy (SPEC acceptance): E2 <= 1e-13 at m = 8."""
    c = case("d1_m8")
    f = oracle.trafo(c["N"], c["n"], 8, c["x"], c["fhat"])
    assert oracle.error_e2(oracle.ndft(c["N"], c["x"], c["fhat"]), f) < 1e-13


def test_oracle_adjoint_blockwise_equals_sequential(oracle):
    c = case("d2_m8")
    a = oracle.adjoint(c["N"], c["n"], 8, c["x"], c["f"], blockwise=True, threads=4)
    b = oracle.adjoint(c["N"], c["n"], 8, c["x"], c["f"], blockwise=False)
    assert oracle.error_e2(b, a) < 1e-14


# ----------------------------------------------------------- scalar pins
def test_pin_gather_ranges():
    """Reference test_indexing.py:50-61 golden values."""
    from paper_1810_09891_b200 import indexing

    r = indexing.gather_range((0.1,), (16,), 2)
    assert [r.lo[0], r.hi[0]] == list(PINS["gr_interior"])
    r = indexing.gather_range((-0.5,), (16,), 2)
    assert [r.lo[0], r.hi[0]] == list(PINS["gr_left"])
    assert r.cells(0, 16).tolist() == PINS["gr_left_cells"].tolist()
    r = indexing.gather_range((0.0,), (8,), 1)
    assert [r.lo[0], r.hi[0]] == list(PINS["gr_centered"])


@pytest.mark.parametrize("d", [1, 2, 3])
def test_pin_node_ranges(oracle, d):
    n = {1: (32,), 2: (16, 12), 3: (16, 16, 16)}[d]
    m = {1: 4, 2: 3, 3: 6}[d]
    lo, width = oracle.node_ranges(n, m, PINS[f"ranges_x_{d}"])
    assert np.array_equal(lo, PINS[f"ranges_lo_{d}"])
    assert np.array_equal(width, PINS[f"ranges_w_{d}"])


def test_pin_bessel_i0(oracle):
    got = np.array([oracle.bessel_i0(v) for v in PINS["i0_x"]])
    assert np.array_equal(got, PINS["i0"])


@pytest.mark.parametrize("kind", ["kaiserbessel", "gaussian"])
@pytest.mark.parametrize("cfg", [(16, 32, 4), (1024, 2048, 8), (64, 128, 6), (256, 512, 4), (16, 20, 3)])
def test_pin_window(oracle, kind, cfg):
    N, n, m = cfg
    key = f"{kind}_{N}_{n}_{m}"
    code = 1 if kind == "gaussian" else 0
    b = oracle.window_b(code, N, n, m)
    assert b == PINS["b_" + key][0]
    phat = [oracle.phi_hat(code, k, n, m, b) for k in range(-N // 2, N // 2 + 1)]
    assert np.allclose(phat, PINS["phihat_" + key], rtol=1e-15, atol=0)
    phi = [oracle.window_factor(code, t, n, m, b) for t in PINS["phi_t_" + key]]
    assert np.allclose(phi, PINS["phi_" + key], rtol=2e-15, atol=0)


def test_pin_kb_edge_limit(oracle):
    """Reference test_window.py:44-48: phi(m/n) = b/pi exactly on the u == 0 branch."""
    b = oracle.window_b(0, 16, 32, 4)
    assert oracle.window_factor(0, 4 / 32, 32, 4, b) == b / np.pi


# --- the reference's own property pins, restated (test_fft.py:31-86,
# test_window.py:147-186): the oracle's FFT against numpy, and the closed-form
# phi_hat against quadrature of the window it transforms.
@pytest.mark.parametrize("shape", [(16,), (514,), (8, 12), (6, 10, 4), (32, 34)])
@pytest.mark.parametrize("sign", [-1, +1])
def test_oracle_fft_matches_numpy(oracle, shape, sign):
    """Unnormalised separable FFT, both signs; radix-2 and Bluestein lengths
    (fft.py:63-139)."""
    rng = np.random.default_rng(7)
    a = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    ref = np.fft.fftn(a) if sign < 0 else np.fft.ifftn(a) * a.size
    out = oracle.fft_nd(a, sign)
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-13


@pytest.mark.parametrize("kind,N,n,m", [("kaiserbessel", 16, 32, 4), ("kaiserbessel", 64, 128, 6),
                                        ("kaiserbessel", 32, 64, 8), ("gaussian", 16, 32, 4),
                                        ("gaussian", 64, 128, 6)])
def test_oracle_phi_hat_matches_quadrature(oracle, kind, N, n, m):
    """phi_hat(k) (window.py:142-164) is the Fourier integral of the window
    (the reference gates the closed forms at 1e-8 against its quadrature
    oracle).  Kaiser-Bessel is integrated over its support |t| <= m/n only:
    the window's sin-branch tail beyond it carries < 1e-8 of the integral for
    m >= 4 (3e-7 at m = 3)."""
    from scipy.integrate import quad

    code = 1 if kind == "gaussian" else 0
    b = oracle.window_b(code, N, n, m)
    lim = m / n if code == 0 else 40.0 * np.sqrt(b) / n
    for k in (0, 1, N // 4, N // 2 - 1, -N // 2):
        val, _ = quad(lambda t: oracle.window_factor(code, t, n, m, b) * np.cos(2 * np.pi * k * t),
                      -lim, lim, limit=400, epsabs=0, epsrel=1e-12)
        ph = oracle.phi_hat(code, k, n, m, b)
        assert abs(val - ph) <= 1e-8 * abs(ph), (k, val, ph)
