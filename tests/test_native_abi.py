"""CPU-side checks of the C ABI: the library loads and exports every symbol
include/poreflow_b200.h declares; argument validation paths that need no GPU."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "poreflow_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(pf_\w+)\(", text, flags=re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for must in ("pf_plan_create", "pf_stokes_solve", "pf_transport_solve", "pf_permeability",
                 "pf_diffusivity", "pf_k_stokes_velocity_update", "pf_k_transport_mode_update", "pf_last_error"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2312_15554_b200 import _native

    lib = _native.load()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(_native.SIGNATURES), "ctypes table out of sync with the header"
    assert lib.pf_version() >= 100


def test_plan_create_rejects_bad_arguments_without_gpu():
    from paper_2312_15554_b200 import _native as N

    lib = N.load()
    h = ctypes.c_void_p()
    assert lib.pf_plan_create(ctypes.byref(h), 4, N.i64_array([8, 8, 8, 8]), 1, 0, None) == N.PF_ERR_ARG
    assert b"ndim" in lib.pf_last_error()
    assert lib.pf_plan_create(ctypes.byref(h), 3, N.i64_array([8, 3, 8]), 1, 0, None) == N.PF_ERR_ARG
    assert lib.pf_plan_create(ctypes.byref(h), 3, N.i64_array([8, 8, 8]), 7, 0, None) == N.PF_ERR_ARG
    with pytest.raises(ValueError):
        N.check(N.PF_ERR_ARG)


def test_solvers_fail_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2312_15554_b200 as pf

    ind = pf.make_model_geometry(pf.UnitCellGrid((8, 8, 8)))
    with pytest.raises(RuntimeError, match="CUDA"):
        pf.solve_stokes(ind, pf.StokesConfig(pressure_gradient=(1.0, 0.0, 0.0)))
    with pytest.raises(RuntimeError, match="CUDA"):
        pf.solve_transport(ind, 0.0 * ind.grid.zeros_vector(), pf.TransportConfig(composition_gradient=(1, 0, 0)))
