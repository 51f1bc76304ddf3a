"""ctypes front end of the CPU oracle (``liboracle.so``).

TEST INFRASTRUCTURE ONLY: imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (cpu_baseline / ``--impl reference``) as the checker.  The
product package ``paper_1810_09891_b200`` never imports this module.

Every entry point restates the reference algorithm (``/root/reference/pkg/
src/nfftk``); see the file:line citations in ``nfft_oracle.c``.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

KAISER_BESSEL = 0
GAUSSIAN = 1
MODE_DIRECT = 0
MODE_LUT = 2


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i32p = ctypes.POINTER(ctypes.c_int)
        vp = ctypes.c_void_p
        L.oracle_trafo.argtypes = [ctypes.c_int, i32p, i32p, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int, ctypes.c_int64, vp, vp, vp]
        L.oracle_adjoint.argtypes = [ctypes.c_int, i32p, i32p, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int64, vp, vp, vp, ctypes.c_int,
                                     ctypes.c_int]
        L.oracle_spread_grid.argtypes = [ctypes.c_int, i32p, i32p, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int64, vp, vp, vp, ctypes.c_int,
                                         ctypes.c_int]
        L.oracle_plan_create.argtypes = [ctypes.c_int, i32p, i32p, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int64, vp]
        L.oracle_plan_create.restype = vp
        L.oracle_plan_destroy.argtypes = [vp]
        L.oracle_plan_destroy.restype = None
        L.oracle_plan_trafo.argtypes = [vp, vp, vp]
        L.oracle_plan_adjoint.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_int]
        L.oracle_gather_grid.argtypes = [ctypes.c_int, i32p, i32p, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int64, vp, vp, vp]
        L.oracle_adjoint_finish.argtypes = [ctypes.c_int, i32p, i32p, ctypes.c_int, ctypes.c_int,
                                            vp, vp]
        L.oracle_ndft.argtypes = [ctypes.c_int, i32p, ctypes.c_int64, vp, vp, vp]
        L.oracle_ndft_adjoint.argtypes = [ctypes.c_int, i32p, ctypes.c_int64, vp, vp, vp]
        L.oracle_fft_nd.argtypes = [ctypes.c_int, i32p, vp, ctypes.c_int]
        L.oracle_node_order.argtypes = [ctypes.c_int, i32p, ctypes.c_int64, vp, vp]
        L.oracle_node_ranges.argtypes = [ctypes.c_int, i32p, ctypes.c_int, ctypes.c_int64, vp, vp, vp]
        L.oracle_window_factor.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double]
        L.oracle_window_factor.restype = ctypes.c_double
        L.oracle_bessel_i0.argtypes = [ctypes.c_double]
        L.oracle_bessel_i0.restype = ctypes.c_double
        L.oracle_phi_hat.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_double]
        L.oracle_phi_hat.restype = ctypes.c_double
        L.oracle_window_b.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.oracle_window_b.restype = ctypes.c_double
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_set_threads.restype = None
        _lib = L
    return _lib


def _ivec(v):
    v = [int(a) for a in v]
    return (ctypes.c_int * len(v))(*v)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _kind(window):
    return GAUSSIAN if str(window).lower() == "gaussian" else KAISER_BESSEL


class Plan:
    """The reference plan's node state and tables (plan.py:202-299: stencils,
    lexicographic order, PRE_PSI factor table) built once; ``trafo`` /
    ``adjoint`` then read them, as the reference's transforms do under its
    default flags (the CPU baseline times only the transforms, like the
    reference's time_mean10 protocol, metrics.py:59-67)."""

    def __init__(self, N, n, m, x, window="kaiserbessel", lut=False):
        self.x = np.ascontiguousarray(x, dtype=np.float64)
        self.M, self.d = self.x.shape
        self.N, self.n, self.m = tuple(int(v) for v in N), tuple(int(v) for v in n), int(m)
        self._h = lib().oracle_plan_create(self.d, _ivec(N), _ivec(n), self.m, _kind(window),
                                           MODE_LUT if lut else MODE_DIRECT, self.M, _ptr(self.x))
        if not self._h:
            raise MemoryError("oracle_plan_create failed (d <= 3, host memory)")

    def trafo(self, fhat, out=None):
        fhat = np.ascontiguousarray(fhat, dtype=np.complex128).ravel()
        out = np.empty(self.M, dtype=np.complex128) if out is None else out
        if lib().oracle_plan_trafo(self._h, _ptr(fhat), _ptr(out)):
            raise MemoryError("oracle_plan_trafo failed")
        return out

    def adjoint(self, f, out=None, blockwise=None, threads=0):
        if blockwise is None:
            blockwise = self.d > 1
        f = np.ascontiguousarray(f, dtype=np.complex128).ravel()
        out = np.empty(int(np.prod(self.N)), dtype=np.complex128) if out is None else out
        if lib().oracle_plan_adjoint(self._h, _ptr(f), _ptr(out), int(bool(blockwise)), int(threads)):
            raise MemoryError("oracle_plan_adjoint failed")
        return out

    def close(self):
        if self._h:
            lib().oracle_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def trafo(N, n, m, x, fhat, window="kaiserbessel", lut=False):
    """Reference trafo (transform.py:92-118) on the CPU."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    M, d = x.shape
    fhat = np.ascontiguousarray(fhat, dtype=np.complex128).ravel()
    out = np.empty(M, dtype=np.complex128)
    rc = lib().oracle_trafo(d, _ivec(N), _ivec(n), int(m), _kind(window),
                            MODE_LUT if lut else MODE_DIRECT, M, _ptr(x), _ptr(fhat), _ptr(out))
    if rc:
        raise ValueError("oracle_trafo supports d <= 3")
    return out


def adjoint(N, n, m, x, f, window="kaiserbessel", lut=False, blockwise=None, threads=0):
    """Reference adjoint (transform.py:121-176) on the CPU."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    M, d = x.shape
    if blockwise is None:
        blockwise = d > 1  # plan.py:77-83 default flag word
    f = np.ascontiguousarray(f, dtype=np.complex128).ravel()
    out = np.empty(int(np.prod(N)), dtype=np.complex128)
    rc = lib().oracle_adjoint(d, _ivec(N), _ivec(n), int(m), _kind(window),
                              MODE_LUT if lut else MODE_DIRECT, M, _ptr(x), _ptr(f), _ptr(out),
                              int(bool(blockwise)), int(threads))
    if rc:
        raise ValueError("oracle_adjoint supports d <= 3")
    return out


def spread_grid(N, n, m, x, f, window="kaiserbessel", lut=False, blockwise=None, threads=0):
    """B^H only (transform.py:121-171): the spread n-grid before the FFT."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    M, d = x.shape
    if blockwise is None:
        blockwise = d > 1
    f = np.ascontiguousarray(f, dtype=np.complex128).ravel()
    g = np.empty(int(np.prod(n)), dtype=np.complex128)
    rc = lib().oracle_spread_grid(d, _ivec(N), _ivec(n), int(m), _kind(window),
                                  MODE_LUT if lut else MODE_DIRECT, M, _ptr(x), _ptr(f), _ptr(g),
                                  int(bool(blockwise)), int(threads))
    if rc:
        raise ValueError("oracle_spread_grid supports d <= 3")
    return g


def gather_grid(N, n, m, x, grid, window="kaiserbessel", lut=False):
    """B alone (kernels.py:122-197): samples at x from a given oversampled grid."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    M, d = x.shape
    g = np.ascontiguousarray(grid, dtype=np.complex128).ravel()
    out = np.empty(M, dtype=np.complex128)
    rc = lib().oracle_gather_grid(d, _ivec(N), _ivec(n), int(m), _kind(window),
                                  MODE_LUT if lut else MODE_DIRECT, M, _ptr(x), _ptr(g), _ptr(out))
    if rc:
        raise ValueError("oracle_gather_grid supports d <= 3")
    return out


def adjoint_finish(N, n, m, grid, window="kaiserbessel"):
    """F^H + D^H of a spread grid (transform.py:174-176)."""
    g = np.array(grid, dtype=np.complex128, copy=True).ravel()
    out = np.empty(int(np.prod(N)), dtype=np.complex128)
    rc = lib().oracle_adjoint_finish(len(N), _ivec(N), _ivec(n), int(m), _kind(window), _ptr(g), _ptr(out))
    if rc:
        raise ValueError("oracle_adjoint_finish supports d <= 3")
    return out


def ndft(N, x, fhat):
    x = np.ascontiguousarray(x, dtype=np.float64)
    M, d = x.shape
    fhat = np.ascontiguousarray(fhat, dtype=np.complex128).ravel()
    out = np.empty(M, dtype=np.complex128)
    lib().oracle_ndft(d, _ivec(N), M, _ptr(x), _ptr(fhat), _ptr(out))
    return out


def ndft_adjoint(N, x, f):
    x = np.ascontiguousarray(x, dtype=np.float64)
    M, d = x.shape
    f = np.ascontiguousarray(f, dtype=np.complex128).ravel()
    out = np.empty(int(np.prod(N)), dtype=np.complex128)
    lib().oracle_ndft_adjoint(d, _ivec(N), M, _ptr(x), _ptr(f), _ptr(out))
    return out


def fft_nd(a, sign):
    a = np.array(a, dtype=np.complex128, order="C", copy=True)
    lib().oracle_fft_nd(a.ndim, _ivec(a.shape), _ptr(a), int(sign))
    return a


def node_order(n, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    M, d = x.shape
    out = np.empty(M, dtype=np.int64)
    lib().oracle_node_order(d, _ivec(n), M, _ptr(x), _ptr(out))
    return out


def node_ranges(n, m, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    M, d = x.shape
    lo = np.empty((M, d), dtype=np.int64)
    width = np.empty((M, d), dtype=np.int64)
    lib().oracle_node_ranges(d, _ivec(n), int(m), M, _ptr(x), _ptr(lo), _ptr(width))
    return lo, width


def window_factor(kind, t, n_i, m, b_i):
    return lib().oracle_window_factor(kind, float(t), float(n_i), float(m), float(b_i))


def bessel_i0(x):
    return lib().oracle_bessel_i0(float(x))


def phi_hat(kind, k, n_i, m, b_i):
    return lib().oracle_phi_hat(kind, int(k), int(n_i), int(m), float(b_i))


def window_b(kind, N_i, n_i, m):
    return lib().oracle_window_b(kind, int(N_i), int(n_i), int(m))


def max_threads():
    return lib().oracle_max_threads()


def set_threads(n):
    """OpenMP threads for the oracle's parallel loops (0 / negative: unchanged)."""
    lib().oracle_set_threads(int(n))


def error_e2(ref, approx):
    """metrics.py:25-34 -- relative l2 error."""
    ref = np.asarray(ref, dtype=np.complex128).ravel()
    approx = np.asarray(approx).astype(np.complex128).ravel()
    return float(np.linalg.norm(ref - approx) / np.linalg.norm(ref))
