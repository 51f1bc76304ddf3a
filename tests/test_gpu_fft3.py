"""Parity of the pruned three-pass F / F^H (csrc/fft.cu: hand-written line
FFTs over the N-band with D, D^H and the ghost padding fused in) against the
CPU oracle and against the cuFFT path of the same plan (NFFTK_NO_PRUNED_FFT).

Covers every supported line length (64..512), mixed lengths per dim, every
radix schedule (8-8, 8-4-4, 8-8-4, 8-8-8), bandwidths other than n/2 (down to
N = 2 and up to the largest whose scratch fits the grid buffer), both
precisions, and the fallbacks (odd geometry -> cuFFT).
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


def run(N, n, m, M, precision, seed=3):
    rng = np.random.default_rng(seed)
    x = rng.random((M, len(N))) - 0.5
    x[0] = -0.5  # halo wrap in every dim: reads the ghost layers the last pass writes
    x[1] = np.nextafter(0.5, 0.0)
    K = int(np.prod(N))
    fh = rng.standard_normal(K) + 1j * rng.standard_normal(K)
    fs = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    p = nf.Plan(N, M, n=n, m=m, precision=precision)
    p.x = x
    p.precompute()
    out = p.fft, p.trafo(fh), p.adjoint(fs)
    p.close()
    return x, fh, fs, out


CASES = [
    # N, n, m
    ((32, 32, 32), (64, 64, 64), 4),
    ((64, 64, 64), (128, 128, 128), 6),
    ((32, 64, 128), (64, 128, 256), 3),
    ((128, 32, 64), (256, 64, 128), 4),
    ((16, 16, 256), (64, 64, 512), 2),
    ((48, 20, 80), (128, 64, 256), 4),   # N != n / 2
    ((20, 48, 36), (64, 128, 256), 4),   # N_2 only a multiple of the half line group (c128) -> skewed layout
    ((2, 2, 16), (64, 64, 64), 2),       # narrowest band
    ((40, 40, 32), (64, 64, 64), 4),     # sigma < 2, scratch still fits
]


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("N,n,m", CASES)
def test_pruned_fft_matches_oracle(N, n, m, precision, oracle):
    M = 3000
    x, fh, fs, (path, f, a) = run(N, n, m, M, precision)
    assert path == ("cufft" if precision == "single" and N[2] % 8 else "pruned")
    assert e2(oracle.trafo(N, n, m, x, fh), f) < TOL[precision]
    assert e2(oracle.adjoint(N, n, m, x, fs), a) < TOL[precision]


@pytest.mark.parametrize("group", ["full", "half"])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_pruned_fft_matches_cufft_path(precision, group, monkeypatch):
    N, n, m, M = (64, 32, 128), (128, 64, 256), 4, 20000
    monkeypatch.delenv("NFFTK_NO_PRUNED_FFT", raising=False)
    monkeypatch.setenv("NFFTK_FFT_G", group)
    _, _, _, (path, f, a) = run(N, n, m, M, precision)
    assert path == "pruned"
    monkeypatch.setenv("NFFTK_NO_PRUNED_FFT", "1")
    _, _, _, (path0, f0, a0) = run(N, n, m, M, precision)
    assert path0 == "cufft"
    tol = 1e-13 if precision == "double" else 2e-6
    assert e2(f0, f) < tol
    assert e2(a0, a) < tol


@pytest.mark.parametrize("N,n", [((24, 24, 24), (48, 48, 48)),      # not a power of two
                                 ((16, 16, 16), (32, 32, 32)),      # below the shortest line
                                 ((60, 60, 60), (64, 64, 64)),      # scratch larger than the grid
                                 ((32, 32, 34), (64, 64, 128))])    # N_2 not a multiple of the (half) line group
def test_unsupported_geometry_takes_cufft(N, n, oracle):
    x, fh, fs, (path, f, a) = run(N, n, 3, 2000, "double")
    assert path == "cufft"
    assert e2(oracle.trafo(N, n, 3, x, fh), f) < 1e-12
    assert e2(oracle.adjoint(N, n, 3, x, fs), a) < 1e-12


def test_repeated_and_chained_transforms(oracle):
    """The trafo's scratch lives in the dense grid buffer and the adjoint's in
    the padded one: alternating calls must not see each other's leftovers."""
    N, n, m, M = (32, 32, 32), (64, 64, 64), 4, 5000
    rng = np.random.default_rng(11)
    x = rng.random((M, 3)) - 0.5
    fh = rng.standard_normal(32 ** 3) + 1j * rng.standard_normal(32 ** 3)
    fs = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    p = nf.Plan(N, M, n=n, m=m)
    p.x = x
    p.precompute()
    assert p.fft == "pruned"
    f_ref = oracle.trafo(N, n, m, x, fh)
    a_ref = oracle.adjoint(N, n, m, x, fs)
    for _ in range(3):
        assert e2(f_ref, p.trafo(fh)) < 1e-12
        assert e2(a_ref, p.adjoint(fs)) < 1e-12
        assert e2(a_ref, p.adjoint(fs)) < 1e-12
        assert e2(f_ref, p.trafo(fh)) < 1e-12
    p.close()


CASES_2D = [
    ((256, 256), (512, 512), 8),     # C2
    ((32, 64), (64, 256), 4),
    ((128, 16), (256, 64), 6),
    ((40, 24), (64, 64), 3),         # sigma < 2
    ((2, 8), (64, 128), 2),
]


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("N,n,m", CASES_2D)
def test_pruned_fft_d2_matches_oracle(N, n, m, precision, oracle):
    """d = 2: two passes (dim 0 on the band columns, dim 1 on all rows into
    the padded grid; the adjoint in reverse)."""
    M = 3000
    x, fh, fs, (path, f, a) = run(N, n, m, M, precision)
    assert path == "pruned"
    assert e2(oracle.trafo(N, n, m, x, fh), f) < TOL[precision]
    assert e2(oracle.adjoint(N, n, m, x, fs), a) < TOL[precision]


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("N,n", [((512, 32), (1024, 64)), ((32, 512), (64, 1024)), ((1024, 16), (2048, 64)),
                                 ((16, 1024), (64, 2048)), ((2048, 8), (4096, 64)), ((8, 2048), (64, 4096)),
                                 ((1000, 24), (2048, 64))])
def test_pruned_fft_d2_long_lines(N, n, precision, oracle):
    """Lines of 1024..4096 (four radix stages; strided groups of 8 / 4 / 2
    lines on the skewed layout, one or two lines per CTA in the contiguous
    pass), as dim 0 and as dim 1."""
    m, M = 4, 3000
    x, fh, fs, (path, f, a) = run(N, n, m, M, precision)
    assert path == "pruned"
    assert e2(oracle.trafo(N, n, m, x, fh), f) < TOL[precision]
    assert e2(oracle.adjoint(N, n, m, x, fs), a) < TOL[precision]


def test_pruned_fft_d3_long_line(oracle):
    N, n, m, M = (16, 512, 8), (64, 1024, 64), 3, 2000
    x, fh, fs, (path, f, a) = run(N, n, m, M, "double")
    assert path == "pruned"
    assert e2(oracle.trafo(N, n, m, x, fh), f) < 1e-12
    assert e2(oracle.adjoint(N, n, m, x, fs), a) < 1e-12


def test_pruned_fft_d2_longer_lines_take_cufft(oracle):
    N, n, m = (4096, 16), (8192, 64), 4
    x, fh, fs, (path, f, a) = run(N, n, m, 2000, "double")
    assert path == "cufft"
    assert e2(oracle.trafo(N, n, m, x, fh), f) < 1e-12
    assert e2(oracle.adjoint(N, n, m, x, fs), a) < 1e-12


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("N,n,m", [((1024,), (2048,), 8), ((32,), (64,), 4), ((100,), (128,), 6),
                                   ((2048,), (4096,), 3), ((2,), (512,), 2)])
def test_pruned_fft_d1_matches_oracle(N, n, m, precision, oracle):
    """d = 1: one fused pass each way (f_hat -> padded grid, grid -> f_hat)."""
    M = 3000
    x, fh, fs, (path, f, a) = run(N, n, m, M, precision)
    assert path == "pruned"
    assert e2(oracle.trafo(N, n, m, x, fh), f) < TOL[precision]
    assert e2(oracle.adjoint(N, n, m, x, fs), a) < TOL[precision]
