"""ctypes binding of ``libporeflow_b200.so`` (include/poreflow_b200.h).

The library is the only compute path of this package: if it is missing or no
CUDA device is visible, every solver entry point raises instead of falling
back to a CPU implementation.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libporeflow_b200.so"

PF_OK, PF_ERR_ARG, PF_ERR_CUDA, PF_ERR_CUFFT, PF_ERR_STATE = 0, 1, 2, 3, 4
PF_SYMBOLS_EXACT, PF_SYMBOLS_CENTRAL = 0, 1

c_double3 = ctypes.c_double * 3


class StokesParams(ctypes.Structure):
    _fields_ = [
        ("nu", ctypes.c_double),
        ("pressure_gradient", c_double3),
        ("eps_abs", ctypes.c_double),
        ("eps_rel", ctypes.c_double),
        ("max_iter", ctypes.c_int64),
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("b", ctypes.c_double),
        ("adaptive", ctypes.c_int32),
        ("growth", c_double3),
        ("ratio_threshold", c_double3),
        ("floor", c_double3),
    ]


class StokesResult(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int64),
        ("converged", ctypes.c_int32),
        ("done", ctypes.c_int32),
        ("final_penalties", c_double3),
    ]


class TransportParams(ctypes.Structure):
    _fields_ = [
        ("pe", ctypes.c_double),
        ("eta", ctypes.c_double),
        ("a0", ctypes.c_double),
        ("b0", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("composition_gradient", c_double3),
        ("max_iter", ctypes.c_int64),
    ]


class TransportResult(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int64),
        ("converged", ctypes.c_int32),
        ("diverged", ctypes.c_int32),
        ("reason", ctypes.c_int32),
        ("done", ctypes.c_int32),
        ("b0_vec", c_double3),
        ("u_bar", c_double3),
    ]


_P = ctypes.c_void_p
_I64P = ctypes.POINTER(ctypes.c_int64)
_DP = ctypes.POINTER(ctypes.c_double)

# name -> argtypes (all return int status except pf_last_error / pf_version)
SIGNATURES = {
    "pf_version": [],
    "pf_last_error": [],
    "pf_plan_create": [ctypes.POINTER(_P), ctypes.c_int, _I64P, ctypes.c_int, ctypes.c_int, _P],
    "pf_plan_destroy": [_P],
    "pf_plan_set_stream": [_P, _P],
    "pf_plan_set_fused": [_P, ctypes.c_int],
    "pf_plan_set_compact": [_P, ctypes.c_int],
    "pf_plan_set_cold_start": [_P, ctypes.c_int],
    "pf_plan_set_symbol_tables": [_P, ctypes.c_int, _P, _P],
    "pf_plan_device_bytes": [_P, ctypes.POINTER(ctypes.c_size_t)],
    "pf_stokes_solve": [_P, ctypes.POINTER(StokesParams), _P, _P, _P, _P, _P, _P, _P, ctypes.POINTER(StokesResult)],
    "pf_stokes_begin": [_P, ctypes.POINTER(StokesParams), _P, _P, _P, _P, _P, _P, _P],
    "pf_stokes_iterate": [_P, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(StokesResult)],
    "pf_stokes_end": [_P, ctypes.POINTER(StokesResult)],
    "pf_stokes_profile": [_P, ctypes.c_int64, _DP],
    "pf_stokes_pipeline": [_P],
    "pf_slab_plan_create": [ctypes.POINTER(_P), _I64P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P],
    "pf_slab_sizes": [_P, _I64P, _I64P, _I64P],
    "pf_slab_forward": [_P, _P, ctypes.c_int, _P],
    "pf_slab_forward_finish": [_P, _P, ctypes.c_int, _P],
    "pf_slab_inverse": [_P, _P, ctypes.c_int, _P],
    "pf_slab_inverse_finish": [_P, _P, ctypes.c_int, _P],
    "pf_slab_stokes_begin": [_P, ctypes.POINTER(StokesParams), _P, _P, _P, _P, _P, _P, _P],
    "pf_slab_setup": [_P, _P, _P, _P, _P],
    "pf_slab_spectral": [_P, _P, _P, _P, _P],
    "pf_slab_local": [_P, _P, _P],
    "pf_slab_finalize": [_P, _P],
    "pf_slab_form_r": [_P, _P, ctypes.c_int],
    "pf_slab_scale": [_P, _P, _P, ctypes.c_int64, ctypes.c_double],
    "pf_slab_read": [_P, ctypes.POINTER(StokesResult)],
    "pf_slab_fused_sizes": [_P, _I64P, _I64P],
    "pf_slab_fused_bind": [_P, _P, _P, _P, _P],
    "pf_slab_fused_setup": [_P, _P, _P, _P],
    "pf_slab_fused_pk": [_P],
    "pf_slab_fused_rs": [_P, _P],
    "pf_slab_fused_mf": [_P],
    "pf_slab_fused_end": [_P, _P],
    "pf_slab_fused_rs_part": [_P, ctypes.c_int],
    "pf_slab_fused_totals": [_P, _P],
    "pf_slab_fused_mf_part": [_P, ctypes.c_int, ctypes.c_int],
    "pf_slab_fused_set_peers": [_P, _P, _P, _P, _P, ctypes.c_int],
    "pf_unpack_bits": [_P, _P, ctypes.c_int64, _P],
    "pf_slab_grad": [_P, _P, ctypes.c_int, _P],
    "pf_slab_fused_setup_zero": [_P],
    "pf_slab_release_transforms": [_P],
    "pf_slab_gram": [_P, _P, _P, _P],
    "pf_transport_solve": [_P, ctypes.POINTER(TransportParams), _P, _P, _P, _P, _P, ctypes.POINTER(TransportResult)],
    "pf_transport_begin": [_P, ctypes.POINTER(TransportParams), _P, _P, _P, _P, _P, ctypes.POINTER(TransportResult)],
    "pf_transport_iterate": [_P, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(TransportResult)],
    "pf_transport_end": [_P, ctypes.POINTER(TransportResult)],
    "pf_transport_pipeline": [_P],
    "pf_transport_profile": [_P, ctypes.c_int64, _DP],
    "pf_pore_average": [_P, _P, _P, ctypes.c_int, _DP],
    "pf_solid_count": [_P, _P, _I64P],
    "pf_permeability": [_P, _P, ctypes.POINTER(_P), _DP],
    "pf_diffusivity": [_P, _P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.c_double, _DP],
    "pf_k_stokes_velocity_update": [ctypes.c_int, _I64P, _P, _P, _P, ctypes.POINTER(_P), _P, _P, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, _DP, _P, _P],
    "pf_k_aux_velocity_update": [ctypes.c_int, _I64P, _P, _P, _P, _P, ctypes.c_double, ctypes.c_double, _P, _P],
    "pf_k_multiplier_update": [ctypes.c_int, _I64P, _P, _P, _P, _P, _P, ctypes.c_double, ctypes.c_double, _P, _P,
                               _P],
    "pf_k_transport_polarization": [ctypes.c_int, _I64P, _P, _P, _P, _P, ctypes.c_double, _DP, _DP, _P, _P, _P],
    "pf_k_transport_mode_update": [ctypes.c_int, _I64P, _P, _P, ctypes.POINTER(_P), _P, ctypes.c_double, _DP, _P,
                                   _P, _P],
    "pf_k_fftn": [ctypes.c_int, _I64P, ctypes.c_int64, _P, ctypes.c_int, _P, ctypes.c_int, _P],
    "pf_k_ifftn_real": [ctypes.c_int, _I64P, ctypes.c_int64, _P, _P, _P, _P],
    "pf_k_spectral_grad": [ctypes.c_int, _I64P, ctypes.c_int64, ctypes.POINTER(_P), _P, _P, _P],
    "pf_k_spectral_div": [ctypes.c_int, _I64P, ctypes.POINTER(_P), _P, _P, _P, _P],
    "pf_k_scale_modes": [ctypes.c_int64, ctypes.c_int64, _P, ctypes.c_double, _P, _P, _P],
    "pf_k_q_update": [ctypes.c_int64, _P, _P, ctypes.c_double, _P, _P, _P],
    "pf_k_norm": [ctypes.c_int64, _P, _P, _P, ctypes.c_int64, _P, _DP, _P],
    "pf_k_scratch_doubles": [],
}

_lib = None
_lock = threading.Lock()


def load(path: Path | str | None = None):
    """Load (once) and type the native library; raise if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path or os.environ.get("POREFLOW_B200_LIB", LIB_PATH))
        if not p.exists():
            raise ImportError(
                f"poreflow_b200 native library not built: {p} (run `python __graft_entry__.py build`)"
            )
        import torch  # noqa: F401  (load torch's libcufft.so.11 first so the SONAME is shared)

        lib = ctypes.CDLL(str(p))
        for name, argtypes in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = ctypes.c_char_p if name == "pf_last_error" else ctypes.c_int
        _lib = lib
        return lib


def check(status: int) -> None:
    if status == PF_OK:
        return
    msg = _lib.pf_last_error().decode(errors="replace") if _lib else "native library not loaded"
    if status == PF_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"poreflow_b200 error {status}: {msg}")


def i64_array(vals):
    arr = (ctypes.c_int64 * len(vals))(*[int(v) for v in vals])
    return arr


def ptr_array(ptrs):
    return (_P * len(ptrs))(*[ctypes.c_void_p(int(p)) for p in ptrs])


def dbl_array(vals, n=None):
    vals = [float(v) for v in vals]
    n = n or len(vals)
    vals = vals + [0.0] * (n - len(vals))
    return (ctypes.c_double * n)(*vals)
