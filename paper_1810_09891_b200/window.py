"""Window model of a plan: kind, oversampling factors and shape parameters.

The closed forms (Kaiser-Bessel and Gaussian phi, phi_hat, the I0 series;
reference window.py:38-181) are implemented ONCE, in the C library
(csrc/plan.cu host math, csrc/common.cuh device math).  This class keeps the
reference's ``WindowModel`` interface -- ``make`` with its validation, ``b``,
``phi``, ``psi``, ``phi_hat``, ``phi_hat_table``, ``ck`` -- and evaluates
through ``nfftk_window_b`` / ``nfftk_window_values`` / ``nfftk_phi_hat_values``
in batches.  The reference's quadrature oracle ``phi_hat_oracle`` is test
infrastructure and is not part of this package.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import NfftError, ShapeError, WindowDegenerateError

KAISER_BESSEL = 0
GAUSSIAN = 1
WINDOW_CODES = {"kaiserbessel": KAISER_BESSEL, "gaussian": GAUSSIAN}


def kind_code(kind):
    """Library code of a window name (case-insensitive)."""
    try:
        return WINDOW_CODES[str(kind).lower()]
    except KeyError:
        raise NfftError(f"unknown window {kind!r}; use 'kaiserbessel' or 'gaussian'") from None


def bessel_i0(x):
    """The library's I0 power series (window.py:38-53)."""
    return float(_lib.load().nfftk_bessel_i0(float(x)))


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


@dataclass(frozen=True)
class WindowModel:
    """Per-dimension window parameters: sigma_i = n_i / N_i, shape b_i."""

    kind: str
    code: int
    n: tuple
    sigma: tuple
    m: int
    b: tuple = field(default=())

    @classmethod
    def make(cls, kind, N, n, m):
        """Validated model (window.py:91-112 rules and messages)."""
        code = kind_code(kind)
        N, n, m = tuple(map(int, N)), tuple(map(int, n)), int(m)
        if len(N) != len(n):
            raise ShapeError("bandlimit and grid vectors differ in length")
        sigma = tuple(ni / Ni for ni, Ni in zip(n, N))
        bad = [s for s in sigma if not s > 1.0]
        if bad:
            raise NfftError(f"oversampling factor must exceed 1, got sigma={bad[0]}")
        wide = [ni for ni in n if not m / ni < 0.5]
        if wide:
            raise NfftError(f"window support m/n={m}/{wide[0]} must be below 1/2")
        lib = _lib.load()
        b = tuple(float(lib.nfftk_window_b(code, Ni, ni, m)) for Ni, ni in zip(N, n))
        return cls(kind=str(kind).lower(), code=code, n=n, sigma=sigma, m=m, b=b)

    @property
    def d(self):
        return len(self.n)

    def _dim(self, i):
        if i < 0 or i >= self.d:
            raise ShapeError(f"dimension index {i} outside [0, {self.d})")
        return i

    def phi(self, t, i=0):
        """phi_i at offsets t (scalar in, scalar out)."""
        i = self._dim(i)
        arr = np.ascontiguousarray(t, dtype=np.float64)
        flat = arr.reshape(-1)
        out = np.empty_like(flat)
        _lib.load().nfftk_window_values(self.code, float(self.n[i]), self.m, self.b[i], _ptr(flat),
                                        flat.size, _ptr(out))
        return float(out[0]) if arr.ndim == 0 else out.reshape(arr.shape)

    def psi(self, t, i=0):
        """phi_i truncated to its support |t| <= m / n_i."""
        t = np.asarray(t, dtype=np.float64)
        inside = np.abs(t) <= self.m / self.n[self._dim(i)]
        return np.where(inside, self.phi(t, i), 0.0)

    def _phi_hat_many(self, ks, i):
        ks = np.ascontiguousarray(ks, dtype=np.int32)
        over = np.abs(ks) > self.n[i] // 2
        if over.any():
            k = int(ks[over][0])
            raise NfftError(f"|k|={abs(k)} exceeds n/2={self.n[i] // 2}")
        vals = np.empty(ks.size)
        status = np.empty(ks.size, dtype=np.int32)
        _lib.load().nfftk_phi_hat_values(self.code, self.n[i], self.m, self.b[i], _ptr(ks), ks.size,
                                         _ptr(vals), _ptr(status))
        if status.any():
            j = int(np.flatnonzero(status)[0])
            k = int(ks[j])
            if status[j] == 1:
                raise WindowDegenerateError(f"{self.kind} transform vanishes at k={k}")
            raise WindowDegenerateError(f"window transform not positive at k={k}: {vals[j]}")
        return vals

    def phi_hat(self, k, i=0):
        """phi_hat_i(k), strictly positive (window.py:142-164)."""
        return float(self._phi_hat_many([int(k)], self._dim(i))[0])

    def phi_hat_table(self, i=0, kmax=None):
        """phi_hat_i over k = -kmax .. kmax (default n_i / 2)."""
        i = self._dim(i)
        kmax = self.n[i] // 2 if kmax is None else int(kmax)
        return self._phi_hat_many(np.arange(-kmax, kmax + 1), i)

    def ck(self, k):
        """Tensor-product coefficient prod_i phi_hat_i(k_i)."""
        k = np.atleast_1d(np.asarray(k, dtype=np.int64))
        if k.shape[0] != self.d:
            raise ShapeError(f"multi-index has {k.shape[0]} dims, window has {self.d}")
        return float(np.prod([self.phi_hat(int(k[i]), i) for i in range(self.d)]))
