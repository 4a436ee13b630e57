"""Effective permeability / diffusivity on device — drop-in for reference
``poreflow.effective`` (pkg/src/poreflow/effective.py:21-108)."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N
from .device import get_plan, require_cuda, solid_on_device, to_device, torch
from .grid import IndicatorField, porosity
from .spectral import CENTRAL, SpectralSymbols


@dataclass
class EffectiveTensors:
    """effective.py:21-29."""

    permeability: np.ndarray
    diffusivity: np.ndarray
    porosity: float
    u_bar: np.ndarray
    meta: dict = field(default_factory=dict)


def pore_average_device(f_dev, indicator: IndicatorField, device=None):
    dev = require_cuda(device)
    grid = indicator.grid
    scalar = tuple(f_dev.shape) == grid.dims
    ncomp = 1 if scalar else int(f_dev.shape[0])
    if ncomp > 3:
        raise ValueError("pore_average supports up to 3 stacked components")
    plan = get_plan(grid.dims, CENTRAL, dev)
    out = (ctypes.c_double * 3)()
    N.check(N.load().pf_pore_average(plan.bind_stream(), solid_on_device(indicator, dev).data_ptr(),
                                     f_dev.contiguous().data_ptr(), ncomp, out))
    return float(out[0]) if scalar else np.asarray(out[:ncomp])


def pore_average(f, indicator: IndicatorField):
    """effective.py:32-40."""
    dev = require_cuda()
    t = torch()
    return pore_average_device(to_device(f, dev, t.float64), indicator, dev)


def permeability(u_solutions: Sequence, indicator: IndicatorField, symbols: SpectralSymbols | str) -> np.ndarray:
    """effective.py:43-72: K_ij = h^d sum_pore grad u^i : grad u^j with the given symbols."""
    grid = indicator.grid
    d = grid.dim
    if len(u_solutions) != d:
        raise ValueError(f"need {d} unit-flow solutions, got {len(u_solutions)}")
    mode = symbols if isinstance(symbols, str) else symbols.mode
    dev = require_cuda()
    t = torch()
    us = []
    for u in u_solutions:
        if tuple(u.shape) != (d, *grid.dims):
            raise ValueError("velocity solution shape does not match the grid")
        us.append(to_device(u, dev, t.float64))
    plan = get_plan(grid.dims, mode, dev)
    K = (ctypes.c_double * (d * d))()
    N.check(N.load().pf_permeability(plan.bind_stream(), solid_on_device(indicator, dev).data_ptr(),
                                      N.ptr_array([u.data_ptr() for u in us]), K))
    return np.asarray(K[:]).reshape(d, d)


def diffusivity(u_solutions: Sequence, chi_solutions: Sequence, indicator: IndicatorField, pe: float) -> np.ndarray:
    """effective.py:75-108."""
    grid = indicator.grid
    d = grid.dim
    if len(u_solutions) != d or len(chi_solutions) != d:
        raise ValueError(f"need {d} flow and {d} concentration solutions")
    if porosity(indicator) == 0.0:
        raise ValueError("diffusivity undefined: no pore cells")
    dev = require_cuda()
    t = torch()
    us = [to_device(u, dev, t.float64) for u in u_solutions]
    chis = [to_device(c[0], dev, t.float64) for c in chi_solutions]
    gch = [to_device(c[1], dev, t.float64) for c in chi_solutions]
    plan = get_plan(grid.dims, CENTRAL, dev)
    D = (ctypes.c_double * (d * d))()
    N.check(N.load().pf_diffusivity(plan.bind_stream(), solid_on_device(indicator, dev).data_ptr(),
                                    N.ptr_array([u.data_ptr() for u in us]),
                                    N.ptr_array([c.data_ptr() for c in chis]),
                                    N.ptr_array([g.data_ptr() for g in gch]), float(pe), D))
    return np.asarray(D[:]).reshape(d, d)
