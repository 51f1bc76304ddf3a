"""ctypes binding of ``libnfftk.so`` (the C-ABI declared in include/nfftk.h).

The shared library is built in-tree (``python -m paper_1810_09891_b200.build``
or ``__graft_entry__.build()``).  There is no fallback: importing the
package without the library raises, so no silent CPU path can stand in for
the CUDA kernels.
"""

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# NFFTK_LIB: development override (A/B builds of the same sources, tools/build_variant.sh)
LIB_PATH = os.environ.get("NFFTK_LIB") or os.path.join(HERE, "libnfftk.so")

_i32, _i64, _u32, _u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
_vp, _cp, _dp = ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_double)
_i32p, _i64p = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)

# name -> (restype, argtypes); every symbol declared in include/nfftk.h
SIGNATURES = {
    "nfftk_abi_version": (_cp, []),
    "nfftk_create": (_i32, [_i32p, _i32, _i32]),
    "nfftk_create_advanced": (_i32, [_i32p, _i32, _i32, _i32p, _i32, _u32, _u32]),
    "nfftk_set_x": (_i32, [_i32, _vp, _i64]),
    "nfftk_set_fhat": (_i32, [_i32, _vp, _i64]),
    "nfftk_set_f": (_i32, [_i32, _vp, _i64]),
    "nfftk_trafo": (_i32, [_i32]),
    "nfftk_adjoint": (_i32, [_i32]),
    "nfftk_get_f": (_vp, [_i32]),
    "nfftk_get_fhat": (_vp, [_i32]),
    "nfftk_last_error": (_i32, [_i32]),
    "nfftk_last_error_message": (_cp, [_i32]),
    "nfftk_destroy": (_i32, [_i32]),
    "nfftk_ext_version": (_cp, []),
    "nfftk_create_ex": (_i32, [_i32p, _i32, _i32, _i32p, _i32, _i32, _i32, _u32, _i32, _u32,
                               _i32, _i32]),
    "nfftk_last_create_error_kind": (_i32, []),
    "nfftk_last_create_error_message": (_cp, []),
    "nfftk_last_error_kind": (_i32, [_i32]),
    "nfftk_set_nodes": (_i32, [_i32, _vp, _i64]),
    "nfftk_set_nodes_device": (_i32, [_i32, _vp, _i64, _vp]),
    "nfftk_precompute": (_i32, [_i32]),
    "nfftk_precompute_stream": (_i32, [_i32, _vp]),
    "nfftk_set_psi_policy": (_i32, [_i32, _i32]),
    "nfftk_trafo_host": (_i32, [_i32, _vp, _vp]),
    "nfftk_adjoint_host": (_i32, [_i32, _vp, _vp]),
    "nfftk_trafo_device": (_i32, [_i32, _vp, _vp, _vp]),
    "nfftk_adjoint_device": (_i32, [_i32, _vp, _vp, _vp]),
    "nfftk_ndft_host": (_i32, [_i32, _vp, _vp]),
    "nfftk_ndft_adjoint_host": (_i32, [_i32, _vp, _vp]),
    "nfftk_ndft_device": (_i32, [_i32, _vp, _vp, _vp]),
    "nfftk_ndft_adjoint_device": (_i32, [_i32, _vp, _vp, _vp]),
    "nfftk_spread_device": (_i32, [_i32, _vp, _vp]),
    "nfftk_adjoint_finish_device": (_i32, [_i32, _vp, _vp]),
    "nfftk_bind_grid": (_i32, [_i32, _vp, _i64]),
    "nfftk_interp_device": (_i32, [_i32, _vp, _vp]),
    "nfftk_deconv_cols": (_i32, [_i32, _i32, _dp, _i64]),
    "nfftk_get_params": (_i32, [_i32, _i64p, _i32]),
    "nfftk_get_sizes": (_i32, [_i32, _i32p, _i32p, _i32p, _i32]),
    "nfftk_get_window": (_i32, [_i32, _dp, _dp, _i32]),
    "nfftk_phi_hut": (_i32, [_i32, _i32, _dp, _i64]),
    "nfftk_node_order": (_i32, [_i32, _i64p, _i64]),
    "nfftk_window_evals": (_i32, [_i32, _i64p, _i64p]),
    "nfftk_psi_tables": (_i32, [_i32, _vp, _vp, _vp, _vp, _i64]),
    "nfftk_lut_tables": (_i32, [_i32, _vp, _vp, _i64]),
    "nfftk_set_timing": (_i32, [_i32, _i32]),
    "nfftk_phase_times": (_i32, [_i32, _dp, _i64p, _i32, _i32]),
    "nfftk_launch_count": (_u64, []),
    "nfftk_measure_fma_peaks": (_i32, [_dp, _dp]),
    "nfftk_window_b": (ctypes.c_double, [_i32, _i32, _i32, _i32]),
    "nfftk_window_values": (_i32, [_i32, ctypes.c_double, _i32, ctypes.c_double, _vp, _i64, _vp]),
    "nfftk_phi_hat_values": (_i32, [_i32, _i32, _i32, ctypes.c_double, _vp, _i64, _vp, _vp]),
    "nfftk_bessel_i0": (ctypes.c_double, [ctypes.c_double]),
    "nfftk_live_handles": (_i32, []),
    "nfftk_live_buffers": (_i64, []),
}

PHASES = ("deconv", "fft_fwd", "interp", "zero", "spread", "fft_inv", "pack", "h2d", "d2h",
          "pad", "fold", "permute")

_lib = None


def load():
    """Load libnfftk.so; raises ImportError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1810_09891_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def i32_array(values):
    values = [int(v) for v in values]
    return (ctypes.c_int32 * max(1, len(values)))(*values)
