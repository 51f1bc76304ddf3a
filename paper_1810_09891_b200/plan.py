"""Drop-in ``Plan`` of the reference (plan.py:124-327) backed by libnfftk.so.

Same constructor, flag words, defaults, validation order, error classes and
transform entry points as the reference ``nfftk.Plan``; the work runs on the
GPU through the C-ABI (include/nfftk.h).  Inputs may be numpy arrays (host
path: one H2D copy, transform, one D2H copy) or CUDA torch tensors (device
path: zero-copy, ordered on the current torch stream, returns a tensor).
"""

import ctypes
import math

import numpy as np

from . import _lib
from .errors import (InvalidFlagError, NfftError, PlanStateError, ShapeError, raise_kind)
from .indexing import validate_bandlimit
from .window import WindowModel, kind_code

# Transform flag word f1, reference bit assignment (plan.py:31-43).
PRE_PHI_HUT = 1 << 0
FG_PSI = 1 << 1
PRE_LIN_PSI = 1 << 2
PRE_FG_PSI = 1 << 3
PRE_PSI = 1 << 4
PRE_FULL_PSI = 1 << 5
MALLOC_X = 1 << 6
MALLOC_F_HAT = 1 << 7
MALLOC_F = 1 << 8
FFT_OUT_OF_PLACE = 1 << 9
FFTW_INIT = 1 << 10
NFFT_SORT_NODES = 1 << 11
NFFT_OMP_BLOCKWISE_ADJOINT = 1 << 12
_NOOP_F1 = MALLOC_X | MALLOC_F_HAT | MALLOC_F | FFT_OUT_OF_PLACE | FFTW_INIT

# FFT-planner word f2 (plan.py:61-70): accepted and ignored.
FFTW_MEASURE = 0
FFTW_DESTROY_INPUT = 1 << 0
FFTW_UNALIGNED = 1 << 1
FFTW_CONSERVE_MEMORY = 1 << 2
FFTW_EXHAUSTIVE = 1 << 3
FFTW_PRESERVE_INPUT = 1 << 4
FFTW_PATIENT = 1 << 5
FFTW_ESTIMATE = 1 << 6
FFTW_WISDOM_ONLY = 1 << 21

DEFAULT_CUTOFF = 8
DEFAULT_F2 = FFTW_ESTIMATE | FFTW_DESTROY_INPUT
LUT_SIZE = 1 << 14

MODE_FOLLOW_FLAGS = -1
MODE_DIRECT = 0
MODE_TENSOR = 1
MODE_LUT = 2

_PRECISIONS = {"double": 0, "complex128": 0, "c128": 0, "single": 1, "complex64": 1, "c64": 1}


def default_f1(d):
    """Default flags (plan.py:77-83): PRE_PHI_HUT | PRE_PSI | sort + no-op bits,
    plus NFFT_OMP_BLOCKWISE_ADJOINT for d > 1."""
    flags = PRE_PHI_HUT | PRE_PSI | NFFT_SORT_NODES | _NOOP_F1
    if d > 1:
        flags |= NFFT_OMP_BLOCKWISE_ADJOINT
    return flags


def default_n(N):
    """Componentwise 2 ** (ceil(log2 N_i) + 1) (plan.py:86-92)."""
    N = validate_bandlimit(N)
    return tuple(1 << ((v - 1).bit_length() + 1) for v in N)


class PrecomputeTables:
    """What precompute built (reference plan.py:109-121): ``phi_hut``,
    ``psi`` (M, d, 2m+1), ``psi_full_vals`` / ``psi_full_idx`` (M, (2m+1)^d)
    and ``psi_full_counts``, ``lut`` (d, 2^14+1) and ``lut_steps``,
    ``node_order``, ``window_evals``.  Entries the plan's f1 does not request
    are None, as in the reference.

    The transforms read their tables on the device, in their own layouts;
    the host arrays above are materialised on first access (device kernels
    in the reference layout and natural node order, then one copy): at C5
    ``psi`` alone is 14.5 GB, which a caller that never inspects it should not
    pay for.  ``psi_on_device`` / ``lut_on_device`` say what the device holds.
    """

    _LAZY = ("psi", "psi_full_vals", "psi_full_idx", "psi_full_counts", "lut", "lut_steps", "node_order")

    def __init__(self, phi_hut=None, window_evals=0, psi_on_device=False, lut_on_device=False,
                 sources=None):
        self.phi_hut = phi_hut
        self.window_evals = window_evals
        self.psi_on_device = psi_on_device
        self.lut_on_device = lut_on_device
        self._sources = dict(sources or {})

    def __getattr__(self, name):
        if name in PrecomputeTables._LAZY:
            src = self.__dict__.get("_sources", {}).pop(name, None)
            value = src() if src is not None else None
            if isinstance(value, dict):  # one source filling several fields
                for k, v in value.items():
                    self.__dict__[k] = v
                    self._sources.pop(k, None)
                return self.__dict__[name]
            self.__dict__[name] = value
            return value
        raise AttributeError(name)

    def __repr__(self):
        return (f"PrecomputeTables(phi_hut={'set' if self.phi_hut is not None else None}, "
                f"lazy={sorted(self._sources)}, window_evals={self.window_evals})")


def _is_torch(a):
    return type(a).__module__.split(".")[0] == "torch"


def _stream_ptr():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class Plan:
    """Reusable transform plan (reference plan.py:124-327) on a B200."""

    def __init__(self, N, M, n=None, m=None, f1=None, f2=None, window="kaiserbessel",
                 precision="double"):
        self._h = 0
        lib = _lib.load()
        self.N = validate_bandlimit(N)
        self.d = len(self.N)
        self.M = int(M)
        nvec = None
        if n is not None:
            try:
                nvec = tuple(int(v) for v in n)
            except TypeError:
                nvec = (int(n),)
            if len(nvec) != self.d:
                raise ShapeError(f"n has {len(nvec)} dims, N has {self.d}")
        if f1 is not None:
            f1 = int(f1)
            if f1 < 0 or f1 != f1 & 0xFFFFFFFF:
                raise InvalidFlagError(f"f1 must be an unsigned 32-bit word, got {f1}")
        prec = _PRECISIONS.get(str(precision).lower())
        if prec is None:
            raise NfftError(f"unknown precision {precision!r}; use 'double' or 'single'")
        try:
            code = kind_code(window)
            bad_window = None
        except NfftError as exc:  # reported after the other checks, as in plan.py:179
            code, bad_window = 0, exc
        h = lib.nfftk_create_ex(
            _lib.i32_array(self.N), self.d, max(-(1 << 31), min(self.M, (1 << 31) - 1)),
            _lib.i32_array(nvec) if nvec is not None else None,
            int(m is not None), int(m) if m is not None else 0,
            int(f1 is not None), (f1 or 0) & 0xFFFFFFFF,
            int(f2 is not None), (int(f2) & 0xFFFFFFFF) if f2 is not None else 0,
            code, prec)
        if h < 0:
            raise_kind(lib.nfftk_last_create_error_kind(),
                       lib.nfftk_last_create_error_message().decode())
        self._h = h
        if bad_window is not None:
            self.close()
            raise bad_window
        self._lib = lib
        self.single = prec == 1
        self.precision = "single" if self.single else "double"
        p = self._params()
        self.m = int(p[2])
        self.f1 = int(p[5])
        self.f2 = int(p[6])
        nn = (ctypes.c_int32 * self.d)()
        tt = (ctypes.c_int32 * self.d)()
        lib.nfftk_get_sizes(h, None, nn, tt, self.d)
        self.n = tuple(int(v) for v in nn)
        self.tile = tuple(int(v) for v in tt)
        self.window = WindowModel.make(window, self.N, self.n, self.m)
        self._x = None
        self._node_order = None
        self._order_valid = False

    # -- plumbing -------------------------------------------------------
    def _params(self):
        out = (ctypes.c_int64 * 16)()
        self._lib_checked().nfftk_get_params(self._h, out, 16)
        return list(out)

    def _lib_checked(self):
        if not self._h:
            raise PlanStateError("plan is closed")
        return _lib.load()

    def _check(self, rc):
        if rc != 0:
            lib = self._lib
            raise_kind(lib.nfftk_last_error_kind(self._h),
                       lib.nfftk_last_error_message(self._h).decode())

    @property
    def handle(self):
        return self._h

    @property
    def cdtype(self):
        return np.complex64 if self.single else np.complex128

    def close(self):
        if self._h:
            _lib.load().nfftk_destroy(self._h)
            self._h = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- sizes ------------------------------------------------------------
    @property
    def num_freqs(self):
        return math.prod(self.N)

    @property
    def grid_size(self):
        return math.prod(self.n)

    # -- nodes (plan.py:202-237) -----------------------------------------
    @property
    def x(self):
        return self._x

    @x.setter
    def x(self, coords):
        self.set_nodes(coords)

    def set_nodes(self, coords):
        """Store the node set (strict [-1/2, 1/2) check, no folding); sorts the
        nodes into grid tiles on the device.  Invalidates precomputed tables."""
        lib = self._lib_checked()
        if _is_torch(coords) and coords.is_cuda:
            import torch

            if tuple(coords.shape) != (self.M, self.d):
                raise ShapeError(f"nodes must have shape {(self.M, self.d)}, got {tuple(coords.shape)}")
            coords = coords.to(torch.float64).contiguous()
            self._check(lib.nfftk_set_nodes_device(self._h, ctypes.c_void_p(coords.data_ptr()),
                                                   coords.numel(), _stream_ptr()))
        else:
            coords = np.asarray(coords, dtype=np.float64)
            if coords.shape != (self.M, self.d):
                raise ShapeError(f"nodes must have shape {(self.M, self.d)}, got {coords.shape}")
            coords = np.ascontiguousarray(coords)
            self._check(lib.nfftk_set_nodes(self._h, coords.ctypes.data, coords.size))
        self._x = coords
        self._order_valid = False

    @property
    def node_order(self):
        """Lexicographic cell order of the nodes when NFFT_SORT_NODES is set
        (plan.py:228-233), computed by a stable device radix sort."""
        if not (self.f1 & NFFT_SORT_NODES) or self._x is None:
            return None
        if not self._order_valid:
            out = np.empty(self.M, dtype=np.int64)
            self._check(self._lib.nfftk_node_order(
                self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), self.M))
            self._node_order = out
            self._order_valid = True
        return self._node_order

    # -- precompute (plan.py:241-299) ------------------------------------
    @property
    def ready(self):
        return bool(self._params()[8])

    def set_psi_policy(self, mode):
        """Extension: force the window-factor source (MODE_DIRECT / MODE_TENSOR)
        regardless of f1; results are identical (kernels.py modes agree)."""
        self._check(self._lib_checked().nfftk_set_psi_policy(self._h, int(mode)))

    def precompute(self):
        lib = self._lib_checked()
        if self._x is not None and _is_torch(self._x):
            self._check(lib.nfftk_precompute_stream(self._h, _stream_ptr()))
        else:
            self._check(lib.nfftk_precompute(self._h))
        return self.tables

    @property
    def tables(self):
        p = self._params()
        if not p[8]:
            return None
        evals = 0
        if self.f1 & (PRE_PSI | PRE_FULL_PSI):
            evals += int(p[12])
        if self.f1 & PRE_LIN_PSI:
            evals += self.d * (LUT_SIZE + 1)
        sources = {"node_order": lambda: self.node_order}
        if self.f1 & (PRE_PSI | PRE_FULL_PSI):
            full = bool(self.f1 & PRE_FULL_PSI)
            fill = lambda: self._psi_tables(full)  # noqa: E731
            for k in (("psi",) if self.f1 & PRE_PSI else ()) + \
                    (("psi_full_vals", "psi_full_idx", "psi_full_counts") if full else ()):
                sources[k] = fill
        if self.f1 & PRE_LIN_PSI:
            sources["lut"] = sources["lut_steps"] = self._lut_tables
        return PrecomputeTables(
            phi_hut=[self.phi_hut(i) for i in range(self.d)] if self.f1 & PRE_PHI_HUT else None,
            window_evals=evals, psi_on_device=p[9] == MODE_TENSOR,
            lut_on_device=bool(self.f1 & PRE_LIN_PSI), sources=sources)

    def _psi_tables(self, full):
        """Reference-layout psi (and PRE_FULL_PSI tables) from the device."""
        K = 2 * self.m + 1
        psi = np.empty((self.M, self.d, K))
        out = {"psi": psi if self.f1 & PRE_PSI else None}
        vals = idx = counts = None
        if full:
            P = K ** self.d
            vals = np.empty((self.M, P))
            idx = np.empty((self.M, P), dtype=np.int64)
            counts = np.empty(self.M, dtype=np.int64)
            out.update(psi_full_vals=vals, psi_full_idx=idx, psi_full_counts=counts)
        ptr = lambda a: ctypes.c_void_p(a.ctypes.data) if a is not None else None  # noqa: E731
        self._check(self._lib_checked().nfftk_psi_tables(self._h, ptr(psi), ptr(vals), ptr(idx),
                                                         ptr(counts), psi.size))
        return out

    def _lut_tables(self):
        lut = np.empty((self.d, LUT_SIZE + 1))
        steps = np.empty(self.d)
        self._check(self._lib_checked().nfftk_lut_tables(self._h, ctypes.c_void_p(lut.ctypes.data),
                                                         ctypes.c_void_p(steps.ctypes.data), lut.size))
        return {"lut": lut, "lut_steps": steps}

    def phi_hut(self, i):
        out = np.empty(self.N[i] + 1)
        self._check(self._lib_checked().nfftk_phi_hut(
            self._h, int(i), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out.size))
        return out

    @property
    def mode(self):
        return int(self._params()[9])

    @property
    def gridding(self):
        """Extension: which gridding kernels a PRE_PSI plan runs -- "residue"
        (residue.cu spread + pipelined interp: d=3, m=4, 8^3 tiles), "pipe"
        (row-per-thread pipelined kernels) or "batch"."""
        return ("batch", "pipe", "residue")[int(self._params()[13])]

    @property
    def fft(self):
        """Extension: how a ready plan runs F / F^H -- "pruned" (fft.cu: three
        passes of line FFTs over the N-band only, with D, D^H and the ghost
        padding fused in; power-of-two n_i of 64..4096) or "cufft" (dense n-grid)."""
        return ("cufft", "pruned")[int(self._params()[15])]

    @property
    def wide_nodes(self):
        """Extension: nodes with a 2m+1 wide stencil in some dim (residue geometry only)."""
        return int(self._params()[14])

    @property
    def window_evals_last(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self._lib_checked().nfftk_window_evals(self._h, ctypes.byref(a), ctypes.byref(b))
        return a.value

    @property
    def window_evals_total(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        self._lib_checked().nfftk_window_evals(self._h, ctypes.byref(a), ctypes.byref(b))
        return b.value

    # -- transforms (transform.py:92-176) ---------------------------------
    def _require_ready(self):
        p = self._params()
        if not p[7]:
            raise PlanStateError("plan has no nodes; call set_nodes() first")
        if not p[8]:
            raise PlanStateError("plan not precomputed; call precompute() first")

    def _as_vector(self, arr, length, what):
        out = np.asarray(arr)
        if out.shape == (length,):
            pass
        elif out.ndim >= 1 and out.size == length:
            out = out.reshape(length)
        else:
            raise ShapeError(f"{what} must have {length} entries, got shape {out.shape}")
        return np.ascontiguousarray(out, dtype=self.cdtype)

    def _as_tensor(self, t, length, what):
        import torch

        if t.numel() != length or t.dim() < 1:
            raise ShapeError(f"{what} must have {length} entries, got shape {tuple(t.shape)}")
        want = torch.complex64 if self.single else torch.complex128
        return t.reshape(length).to(want).contiguous()

    def _check_out_array(self, out, length, what):
        """``out=`` for the host path: the library writes ``length`` elements
        of the plan's complex type at ``out.ctypes.data``."""
        if not isinstance(out, np.ndarray):
            raise ShapeError(f"{what} out= must be a numpy array on the host path")
        if out.dtype != self.cdtype or out.size != length or not out.flags.c_contiguous \
                or not out.flags.writeable:
            raise ShapeError(f"{what} out= must be a writeable C-contiguous {np.dtype(self.cdtype).name} "
                             f"array of {length} entries, got {out.dtype} shape {out.shape}")
        return out

    def _check_out_tensor(self, out, length, what, device):
        """``out=`` for the device path: a contiguous tensor of the plan's
        complex dtype on the input's device."""
        import torch

        want = torch.complex64 if self.single else torch.complex128
        if not (_is_torch(out) and out.is_cuda):
            raise ShapeError(f"{what} out= must be a CUDA tensor on the device path")
        if out.dtype != want or out.numel() != length or not out.is_contiguous() or out.device != device:
            raise ShapeError(f"{what} out= must be a contiguous {want} tensor of {length} entries on "
                             f"{device}, got {out.dtype} shape {tuple(out.shape)} on {out.device}")
        return out

    def trafo(self, fhat, out=None):
        """f = B F D f_hat at the M nodes (transform.py:92-118)."""
        lib = self._lib_checked()
        self._require_ready()
        if _is_torch(fhat) and fhat.is_cuda:
            import torch

            fhat = self._as_tensor(fhat, self.num_freqs, "fhat")
            if out is None:
                out = torch.empty(self.M, dtype=fhat.dtype, device=fhat.device)
            self._check_out_tensor(out, self.M, "trafo", fhat.device)
            self._check(lib.nfftk_trafo_device(self._h, ctypes.c_void_p(fhat.data_ptr()),
                                               ctypes.c_void_p(out.data_ptr()), _stream_ptr()))
            return out
        fhat = self._as_vector(fhat, self.num_freqs, "fhat")
        if out is None:
            out = np.empty(self.M, dtype=self.cdtype)
        self._check_out_array(out, self.M, "trafo")
        self._check(lib.nfftk_trafo_host(self._h, fhat.ctypes.data, out.ctypes.data))
        return out

    def adjoint(self, f, out=None):
        """f_hat = D^H F^H B^H f (transform.py:121-176)."""
        lib = self._lib_checked()
        self._require_ready()
        if _is_torch(f) and f.is_cuda:
            import torch

            f = self._as_tensor(f, self.M, "f")
            if out is None:
                out = torch.empty(self.num_freqs, dtype=f.dtype, device=f.device)
            self._check_out_tensor(out, self.num_freqs, "adjoint", f.device)
            self._check(lib.nfftk_adjoint_device(self._h, ctypes.c_void_p(f.data_ptr()),
                                                 ctypes.c_void_p(out.data_ptr()), _stream_ptr()))
            return out
        f = self._as_vector(f, self.M, "f")
        if out is None:
            out = np.empty(self.num_freqs, dtype=self.cdtype)
        self._check_out_array(out, self.num_freqs, "adjoint")
        self._check(lib.nfftk_adjoint_host(self._h, f.ctypes.data, out.ctypes.data))
        return out

    # -- multi-GPU building blocks (distributed.py) -----------------------
    def spread(self, f):
        """B^H only, into the plan grid (device tensor input)."""
        if not (_is_torch(f) and f.is_cuda):
            raise ShapeError("spread() takes a CUDA tensor")
        f = self._as_tensor(f, self.M, "f")
        self._check(self._lib_checked().nfftk_spread_device(
            self._h, ctypes.c_void_p(f.data_ptr()), _stream_ptr()))

    def interp(self, out=None):
        """B alone: samples at the plan's nodes from its dense grid (a grid
        bound with ``bind_grid`` and filled by the caller -- the slab trafo of
        distributed.py), on the current stream."""
        import torch

        lib = self._lib_checked()
        self._require_ready()
        grid = getattr(self, "_bound_grid", None)
        if grid is None:
            raise PlanStateError("interp() reads a bound grid; call bind_grid() first")
        if out is None:
            out = torch.empty(self.M, dtype=torch.complex64 if self.single else torch.complex128,
                              device=grid.device)
        self._check_out_tensor(out, self.M, "interp", grid.device)
        self._check(lib.nfftk_interp_device(self._h, ctypes.c_void_p(out.data_ptr()), _stream_ptr()))
        return out

    def deconv_cols(self, i):
        """1 / (phi_hat_i(k) * wscale_i) for k = -N_i/2 .. N_i/2 - 1: the
        deconvolution column D applies with 1/|I_n| (transform.py:44-63)."""
        out = np.empty(self.N[i])
        self._check(self._lib_checked().nfftk_deconv_cols(
            self._h, int(i), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), out.size))
        return out

    def adjoint_finish(self, out):
        """F^H and D^H of the (already reduced) plan grid into ``out``."""
        import torch

        self._check_out_tensor(out, self.num_freqs, "adjoint_finish",
                               out.device if _is_torch(out) else torch.device("cuda"))
        self._check(self._lib_checked().nfftk_adjoint_finish_device(
            self._h, ctypes.c_void_p(out.data_ptr()), _stream_ptr()))
        return out

    def bind_grid(self, tensor):
        """Use a caller-owned device tensor as the plan's oversampled grid."""
        if not (_is_torch(tensor) and tensor.is_cuda and tensor.is_contiguous()):
            raise ShapeError("bind_grid() takes a contiguous CUDA tensor")
        nbytes = tensor.numel() * tensor.element_size()
        self._check(self._lib_checked().nfftk_bind_grid(self._h, ctypes.c_void_p(tensor.data_ptr()),
                                                        nbytes))
        self._bound_grid = tensor

    # -- instrumentation ------------------------------------------------
    def set_timing(self, on=True):
        self._lib_checked().nfftk_set_timing(self._h, int(bool(on)))

    def phase_times(self, reset=False):
        """Accumulated CUDA-event milliseconds and call counts per phase."""
        n = len(_lib.PHASES)
        ms = (ctypes.c_double * n)()
        calls = (ctypes.c_int64 * n)()
        self._check(self._lib_checked().nfftk_phase_times(self._h, ms, calls, n, int(bool(reset))))
        return {name: (ms[i], calls[i]) for i, name in enumerate(_lib.PHASES)}

    def _exact(self, data, length, what, outlen, host_fn, dev_fn):
        lib = self._lib_checked()
        if not self._params()[7]:
            raise PlanStateError("plan has no nodes; call set_nodes() first")
        if _is_torch(data) and data.is_cuda:
            import torch

            if data.numel() != length or data.dim() < 1:
                raise ShapeError(f"{what} must have {length} entries, got shape {tuple(data.shape)}")
            data = data.reshape(length).to(torch.complex128).contiguous()
            out = torch.empty(outlen, dtype=torch.complex128, device=data.device)
            self._check(getattr(lib, dev_fn)(self._h, ctypes.c_void_p(data.data_ptr()),
                                             ctypes.c_void_p(out.data_ptr()), _stream_ptr()))
            return out
        out_arr = np.asarray(data)
        if not (out_arr.shape == (length,) or (out_arr.ndim >= 1 and out_arr.size == length)):
            raise ShapeError(f"{what} must have {length} entries, got shape {out_arr.shape}")
        vec = np.ascontiguousarray(out_arr.reshape(length), dtype=np.complex128)
        out = np.empty(outlen, dtype=np.complex128)
        self._check(getattr(lib, host_fn)(self._h, vec.ctypes.data, out.ctypes.data))
        return out

    def ndft(self, fhat):
        """Exact forward sums f_j = sum_k fhat_k e^{-2 pi i k x_j}, O(M |I_N|)
        (transform.py:188-203), on the device; complex128 regardless of the
        plan precision."""
        return self._exact(fhat, self.num_freqs, "fhat", self.M, "nfftk_ndft_host", "nfftk_ndft_device")

    def ndft_adjoint(self, f):
        """Exact adjoint sums fhat_k = sum_j f_j e^{+2 pi i k x_j}
        (transform.py:206-234), on the device; complex128."""
        return self._exact(f, self.M, "f", self.num_freqs, "nfftk_ndft_adjoint_host",
                           "nfftk_ndft_adjoint_device")

    def __repr__(self):
        return (f"Plan(N={self.N}, M={self.M}, n={self.n}, m={self.m}, "
                f"f1={hex(self.f1)}, f2={hex(self.f2)}, window={self.window.kind!r})")


def launch_count():
    """Kernels launched by libnfftk.so in this process."""
    return int(_lib.load().nfftk_launch_count())
