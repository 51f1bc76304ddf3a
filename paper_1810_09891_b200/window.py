"""Window model of a plan (kind, sigma, b) with host evaluators.

Same closed forms as the reference (window.py:56-181): Kaiser-Bessel
phi(t) = sinh(b sqrt(m^2 - (n t)^2)) / (pi sqrt(.)) with b = pi (2 - 1/sigma),
phi_hat(k) = I0(m sqrt(b^2 - (2 pi k / n)^2)) / n; Gaussian
phi(t) = exp(-(n t)^2 / b) / sqrt(pi b), b = 2 sigma m / ((2 sigma - 1) pi),
phi_hat(k) = exp(-b (pi k / n)^2) / n.  These host evaluators serve the
Python API (``plan.window.phi`` ...); the transforms evaluate the window on
the device (csrc/common.cuh) and build phi_hat in the C library.
The quadrature oracle ``phi_hat_oracle`` of the reference is test-only and
not part of this package.
"""

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import NfftError, ShapeError, WindowDegenerateError

KAISER_BESSEL = 0
GAUSSIAN = 1
_KIND_BY_NAME = {"kaiserbessel": KAISER_BESSEL, "gaussian": GAUSSIAN}


def bessel_i0(x):
    """I0 power series, term-ratio cutoff 1e-16 (window.py:38-53)."""
    s = t = 1.0
    q = 0.25 * x * x
    j = 0
    while True:
        j += 1
        t *= q / (j * j)
        s += t
        if t < 1e-16 * s:
            return s


def window_factor(code, t, n_i, m, b_i):
    """Scalar window value at offset t (window.py:56-72)."""
    if code == KAISER_BESSEL:
        u = m * m - (n_i * t) * (n_i * t)
        if u > 0.0:
            z = math.sqrt(u)
            return math.sinh(b_i * z) / (math.pi * z)
        if u < 0.0:
            z = math.sqrt(-u)
            return math.sin(b_i * z) / (math.pi * z)
        return b_i / math.pi
    return math.exp(-(n_i * t) * (n_i * t) / b_i) / math.sqrt(math.pi * b_i)


def kind_code(kind):
    code = _KIND_BY_NAME.get(str(kind).lower())
    if code is None:
        raise NfftError(f"unknown window {kind!r}; use 'kaiserbessel' or 'gaussian'")
    return code


@dataclass(frozen=True)
class WindowModel:
    kind: str
    code: int
    n: tuple
    sigma: tuple
    m: int
    b: tuple = field(default=())

    @classmethod
    def make(cls, kind, N, n, m):
        code = kind_code(kind)
        N = tuple(int(v) for v in N)
        n = tuple(int(v) for v in n)
        m = int(m)
        if len(N) != len(n):
            raise ShapeError("bandlimit and grid vectors differ in length")
        sigma = tuple(ni / Ni for ni, Ni in zip(n, N))
        for s in sigma:
            if s <= 1.0:
                raise NfftError(f"oversampling factor must exceed 1, got sigma={s}")
        for ni in n:
            if m / ni >= 0.5:
                raise NfftError(f"window support m/n={m}/{ni} must be below 1/2")
        if code == KAISER_BESSEL:
            b = tuple(math.pi * (2.0 - 1.0 / s) for s in sigma)
        else:
            b = tuple(2.0 * s * m / ((2.0 * s - 1.0) * math.pi) for s in sigma)
        return cls(kind=str(kind).lower(), code=code, n=n, sigma=sigma, m=m, b=b)

    @property
    def d(self):
        return len(self.n)

    def _dim(self, i):
        if not 0 <= i < self.d:
            raise ShapeError(f"dimension index {i} outside [0, {self.d})")
        return i

    def phi(self, t, i=0):
        i = self._dim(i)
        t = np.asarray(t, dtype=np.float64)
        f = np.vectorize(lambda v: window_factor(self.code, float(v), float(self.n[i]),
                                                 float(self.m), self.b[i]), otypes=[float])
        out = f(t)
        return float(out) if t.ndim == 0 else out

    def psi(self, t, i=0):
        i = self._dim(i)
        t = np.asarray(t, dtype=np.float64)
        return np.where(np.abs(t) <= self.m / self.n[i], self.phi(t, i), 0.0)

    def phi_hat(self, k, i=0):
        i = self._dim(i)
        k = int(k)
        n_i = self.n[i]
        if abs(k) > n_i // 2:
            raise NfftError(f"|k|={abs(k)} exceeds n/2={n_i // 2}")
        if self.code == KAISER_BESSEL:
            arg = self.b[i] ** 2 - (2.0 * math.pi * k / n_i) ** 2
            if arg < 0.0:
                raise WindowDegenerateError(f"kaiserbessel transform vanishes at k={k}")
            val = bessel_i0(self.m * math.sqrt(arg)) / n_i
        else:
            val = math.exp(-self.b[i] * (math.pi * k / n_i) ** 2) / n_i
        if not val > 0.0:
            raise WindowDegenerateError(f"window transform not positive at k={k}: {val}")
        return val

    def phi_hat_table(self, i=0, kmax=None):
        i = self._dim(i)
        if kmax is None:
            kmax = self.n[i] // 2
        return np.array([self.phi_hat(k, i) for k in range(-kmax, kmax + 1)])

    def ck(self, k):
        k = np.atleast_1d(np.asarray(k, dtype=np.int64))
        if k.shape[0] != self.d:
            raise ShapeError(f"multi-index has {k.shape[0]} dims, window has {self.d}")
        out = 1.0
        for i in range(self.d):
            out *= self.phi_hat(int(k[i]), i)
        return out
