"""ctypes binding of libmlb.so (include/multilap_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is present, `lib()` raises.  Device buffers come from torch
(plumbing only); every byte of the hot path runs in libmlb.so's kernels.
"""

import ctypes as C
import os
import threading

from .errors import ConfigError, NumericalError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmlb.so")

MLB_OK, MLB_ERR_CONFIG, MLB_ERR_NUMERICAL, MLB_ERR_CUDA, MLB_ERR_ARG = 0, 1, 2, 3, 4
MLB_USE_ISD, MLB_ACCUMULATE, MLB_SORTED, MLB_SPREAD_ONLY = 1, 2, 4, 8

_lock = threading.Lock()
_lib = None

P = C.c_void_p
D = C.c_double
I = C.c_int
I64 = C.c_int64
U = C.c_uint


class PlanDesc(C.Structure):
    _fields_ = [("d", I), ("N", I), ("m", I), ("ng", I), ("bin_lo", I), ("bin_hi", I),
                ("win_deg", I), ("K0", D), ("fused_band", P), ("twiddle", P), ("win_coef", P),
                ("conv_kernel", P), ("sep_kernel", P)]


class BindDesc(C.Structure):
    """mlb_bind_desc (include/multilap_b200.h)."""
    _fields_ = [("points", P), ("points_on_device", I), ("n", I64), ("ld", I), ("cols", P), ("scale", D),
                ("box_mid", P), ("box_half", D), ("box_s", D), ("box_hw", D), ("node_ids", P), ("stream", P)]


# name -> (restype, argtypes); mirrors include/multilap_b200.h
SIGNATURES = {
    "mlb_abi_version": (I, []),
    "mlb_last_error": (C.c_char_p, []),
    "mlb_device_count": (I, []),
    "mlb_launch_count": (I64, []),
    "mlb_note_launches": (None, [I64]),
    "mlb_probe_fp64": (I, [I64, I, P, P]),
    "mlb_probe_dmma": (I, [I64, I, P, P]),
    "mlb_plan_create": (I, [C.POINTER(PlanDesc), I, C.POINTER(P)]),
    "mlb_plan_destroy": (I, [P]),
    "mlb_bind": (I, [P, P, I64, D, P, C.POINTER(P)]),
    "mlb_bind_ex": (I, [P, C.POINTER(BindDesc), C.POINTER(P)]),
    "mlb_binding_destroy": (I, [P]),
    "mlb_binding_n": (I64, [P]),
    "mlb_binding_perm": (I, [P, P]),
    "mlb_binding_stats": (I, [P, P]),
    "mlb_binding_lattice": (I, [P, P]),
    "mlb_binding_set_isd": (I, [P, P, P]),
    "mlb_apply": (I, [P, P, P, D, D, D, U, P]),
    "mlb_grid_cells": (I, [P, P, P, P]),
    "mlb_spread": (I, [P, P, P, U, P]),
    "mlb_reduce": (I, [P, P, P]),
    "mlb_spread_peers": (I, [P, P, P, I, U, P]),
    "mlb_apply_batched": (I, [P, I, P, P, P, P, P, U, P]),
    "mlb_grid_sum_slots": (I, [P, I, I64, P, P]),
    "mlb_ipc_handle": (I, [P, P]),
    "mlb_ipc_open": (I, [P, I, P]),
    "mlb_ipc_close": (I, [P]),
    "mlb_convolve": (I, [P, P, P, P]),
    "mlb_gather": (I, [P, P, P, U, P]),
    "mlb_gather_apply": (I, [P, P, P, P, D, D, D, U, P]),
    "mlb_band_dft": (I, [P, P, P, I, P]),
    "mlb_to_sorted": (I, [P, P, P, P]),
    "mlb_to_node": (I, [P, P, P, I, P]),
    "mlb_krylov_work_size": (I64, [I64, I]),
    "mlb_gemv_t": (I, [P, I64, I64, I, P, P, P, P]),
    "mlb_cgs2": (I, [P, I64, I64, I, P, P, P, P, P, P]),
    "mlb_gemv_n": (I, [P, I64, I64, I, P, P, D, I, P]),
    "mlb_cgs2_batched_work_size": (I64, [I]),
    "mlb_cgs2_batched": (I, [I, P, I64, I64, I, P, P, P, P, P, P, P]),
    "mlb_tridiag_fn_batched": (I, [I, P, I64, I, I, D, P, P, P]),
    "mlb_apply_multi": (I, [P, I, P, P, P, U, P]),
    "mlb_gemm_vs": (I, [P, I64, I64, I, P, I, P, I64, P]),
    "mlb_dot": (I, [P, P, I64, P, P, P]),
    "mlb_axpby": (I, [D, P, D, P, I64, P]),
    "mlb_scale_by": (I, [P, P, I64, P, D, P]),
    "mlb_hadamard": (I, [P, P, P, I64, P]),
    "mlb_direct": (I, [P, I64, I, I, D, P, P, P, D, D, D, I, P]),
    "mlb_direct_targets_work_size": (I64, [I64]),
    "mlb_direct_targets": (I, [P, I64, I, I, D, P, P, I64, P, P, P]),
    "mlb_ac_work_size": (I64, [I64, I, I]),
    "mlb_ac_step": (I, [P, I64, I, I, P, P, P, P, D, D, D, P, P, P, P]),
    "mlb_argmax_rows": (I, [P, I64, I, P, P]),
    "mlb_ac_step2": (I, [P, I64, I, I, P, P, P, P, D, D, D, I, P, P, P, P]),
    "mlb_ac_rhs_partial": (I, [P, I64, I, I, P, P, P, D, D, D, P, P, P]),
    "mlb_ac_update_from": (I, [P, I64, I, I, P, P, P, P, P, P, P]),
    "mlb_bac_step": (I, [P, I64, I, P, P, P, P, P, D, D, D, P, P, P, P, P]),
    "mlb_gl_energy_work_size": (I64, [I, I]),
    "mlb_gl_energy_partials": (I, [P, I64, I, I, P, P, P, P, P, P]),
}


def _maybe_rebuild():
    """Rebuild libmlb.so when a source is newer and nvcc is available."""
    from . import build as _build
    try:
        stale = _build.needs_build()
    except OSError:
        return
    if stale and os.path.exists(_build.NVCC):
        _build.build()


def load(path=LIB_PATH):
    """Load libmlb.so and declare every exported symbol (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if path == LIB_PATH and os.environ.get("MLB_LIB_VARIANT"):
            # A/B experiments: an alternative in-tree build of the same ABI
            path = os.path.join(_HERE, os.environ["MLB_LIB_VARIANT"])
        elif path == LIB_PATH:
            _maybe_rebuild()
        if not os.path.exists(path):
            raise RuntimeError(
                f"libmlb.so not found at {path}; build it with "
                "`python -m paper_2007_05239_b200.build` (there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            if not hasattr(lib, name):
                continue  # reported by tests/test_capi.py
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib():
    """The loaded library, after checking a CUDA device is usable."""
    L = load()
    if L.mlb_device_count() < 1:
        raise RuntimeError("no CUDA device visible to libmlb.so; the B200 path cannot run")
    return L


def check(rc):
    if rc == MLB_OK:
        return
    msg = (load().mlb_last_error() or b"").decode(errors="replace")
    if rc == MLB_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == MLB_ERR_NUMERICAL:
        raise NumericalError(msg)
    raise RuntimeError(f"libmlb error {rc}: {msg}")


def ptr(t):
    """Raw device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)
