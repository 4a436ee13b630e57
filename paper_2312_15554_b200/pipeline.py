"""Cell-to-tensors pipeline on device — the computational core of the
reference's ``cli.run`` (pkg/src/poreflow/cli.py:282-414) without its file
I/O: d unit-pressure-gradient Stokes solves, the physical flow by
superposition (cli.py:348), d unit-composition-gradient transport solves under
that flow (cli.py:361-371), and K*, D*, porosity, pore-mean velocities
(cli.py:386-408).  Every field stays on the GPU; only the tensors, reports and
(optionally) the physical fields come back to the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from .device import require_cuda, torch
from .effective import EffectiveTensors, diffusivity, permeability, pore_average_device
from .grid import IndicatorField, porosity
from .batch import solve_stokes_many_device, solve_transport_many_device
from .stokes import PenaltyParams, StokesConfig
from .transport import TransportConfig


@dataclass
class CellResult:
    tensors: EffectiveTensors
    flow_reports: list
    transport_reports: list
    u_phys: object = None      # device tensor (d, *dims)
    chi_phys: object = None    # device tensor (*dims)
    meta: dict = field(default_factory=dict)

    @property
    def converged(self) -> bool:
        return all(r.converged for r in self.flow_reports + self.transport_reports)


def _unit(d, axis):
    g = [0.0] * d
    g[axis] = 1.0
    return tuple(g)


def effective_tensors(indicator: IndicatorField, stokes_cfg: StokesConfig | None = None,
                      transport_cfg: TransportConfig | None = None, penalties: PenaltyParams | None = None,
                      device=None) -> CellResult:
    """K*, D* of one periodic cell (cli.run's flow, device-resident)."""
    dev = require_cuda(device)
    grid = indicator.grid
    d = grid.dim
    stokes_cfg = stokes_cfg or StokesConfig(pressure_gradient=_unit(d, 0))
    transport_cfg = transport_cfg or TransportConfig(composition_gradient=_unit(d, 0))
    phi = porosity(indicator)
    if phi == 0.0:
        zeros = np.zeros((d, d))
        return CellResult(EffectiveTensors(zeros, np.full((d, d), np.nan), 0.0, zeros,
                                           meta={"note": "all-solid geometry: zero flow, transport undefined"}),
                          [], [])
    # the d unit solves of each stage are independent: run them concurrently (batch.py)
    flows = solve_stokes_many_device([indicator] * d, [replace(stokes_cfg, pressure_gradient=_unit(d, axis))
                                                       for axis in range(d)], penalties, dev)
    unit_u = [st.u for st, _ in flows]
    flow_reports = [rep for _, rep in flows]
    g_p = np.asarray(stokes_cfg.pressure_gradient, dtype=float)
    u_phys = sum(float(g_p[i]) * unit_u[i] for i in range(d))
    trs = solve_transport_many_device([indicator] * d, [u_phys] * d,
                                      [replace(transport_cfg, composition_gradient=_unit(d, axis)) for axis in range(d)],
                                      dev)
    chis = [(ts.chi, ts.grad_chi) for ts, _ in trs]
    transport_reports = [rep for _, rep in trs]
    g_chi = np.asarray(transport_cfg.composition_gradient, dtype=float)
    chi_phys = sum(float(g_chi[j]) * chis[j][0] for j in range(d))
    K = permeability(unit_u, indicator, stokes_cfg.symbol_mode)
    D = diffusivity(unit_u, chis, indicator, transport_cfg.pe)
    u_bar = np.stack([np.atleast_1d(pore_average_device(u, indicator, dev)) for u in unit_u])
    tensors = EffectiveTensors(
        permeability=K, diffusivity=D, porosity=phi, u_bar=u_bar,
        meta={"nu": stokes_cfg.nu, "flow_tolerance": [stokes_cfg.eps_abs, stokes_cfg.eps_rel],
              "transport_tolerance": transport_cfg.eps, "flow_symbol_mode": stokes_cfg.symbol_mode,
              "transport_symbol_mode": transport_cfg.symbol_mode,
              "flow_iterations": [r.iterations for r in flow_reports],
              "transport_iterations": [r.iterations for r in transport_reports],
              "velocity_convention": "concentration solved under the configured-direction flow; "
                                     "unit flows enter the tensor"})
    torch().cuda.synchronize(dev)
    return CellResult(tensors, flow_reports, transport_reports, u_phys, chi_phys,
                      meta={"u_bar_physical": pore_average_device(u_phys, indicator, dev)})
