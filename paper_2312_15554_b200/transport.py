"""Comparison-medium transport solver on B200 — drop-in for reference
``poreflow.transport`` (pkg/src/poreflow/transport.py).

The loop (transport.py:225-258) runs on device behind ``pf_transport_*``; the
medium coefficients A, B, F are derived per voxel from the indicator and the
velocity inside the fused kernels (build_coefficients, transport.py:101-128,
is still offered for API callers and is computed on device).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .device import get_plan, require_cuda, solid_on_device, to_device, to_host_many, torch
from .grid import IndicatorField
from .report import ConvergenceReport
from .spectral import CENTRAL, SYMBOL_MODES

REPORT_COLUMNS = ("r1", "r1_tol", "r2", "r2_tol")  # transport.py:28
DIVERGENCE_GROWTH = 1e6  # transport.py:32
_REASONS = {
    0: "",
    1: "non-finite residual",
    2: (f"residual grew {DIVERGENCE_GROWTH:.0e}x over its minimum; "
        "comparison diffusivity a0 is below the convergence boundary"),
}


@dataclass
class TransportConfig:
    """transport.py:35-65."""

    pe: float = 0.0
    composition_gradient: tuple = (1.0, 0.0)
    eta: float = 0.01
    a0: float = 0.55
    b0: float = 1.0
    eps: float = 1e-5
    max_iter: int = 10_000
    symbol_mode: str = CENTRAL

    def __post_init__(self):
        if self.pe < 0.0:
            raise ValueError("Peclet number must be nonnegative")
        if not 0.0 < self.eta <= 1.0:
            raise ValueError("fictitious diffusivity eta must lie in (0, 1]")
        if self.a0 <= 0.0:
            raise ValueError("comparison diffusivity a0 must be positive")
        if self.eps <= 0.0:
            raise ValueError("tolerance must be positive")
        if self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")
        if self.symbol_mode not in SYMBOL_MODES:
            raise ValueError(f"symbol_mode must be one of {SYMBOL_MODES}")


@dataclass
class TransportState:
    """transport.py:68-81 (host arrays)."""

    chi: np.ndarray
    grad_chi: np.ndarray
    iterations: int = 0

    @classmethod
    def zeros(cls, grid) -> "TransportState":
        return cls(chi=grid.zeros_scalar(), grad_chi=grid.zeros_vector())

    def copy(self) -> "TransportState":
        return TransportState(self.chi.copy(), self.grad_chi.copy(), self.iterations)


@dataclass
class DeviceTransportState:
    chi: object
    grad_chi: object
    iterations: int = 0

    def to_host(self) -> TransportState:
        chi, gch = to_host_many([self.chi, self.grad_chi])
        return TransportState(chi, gch, self.iterations)


@dataclass(frozen=True)
class MediumCoefficients:
    """transport.py:84-98."""

    diffusivity: np.ndarray
    advection: np.ndarray
    forcing: np.ndarray
    u_bar: np.ndarray
    b0_vec: np.ndarray


def _check_velocity(indicator, u):
    grid = indicator.grid
    if tuple(u.shape) != (grid.dim, *grid.dims):
        raise ValueError("velocity shape does not match the grid")


def build_coefficients(indicator: IndicatorField, u, cfg: TransportConfig) -> MediumCoefficients:
    """transport.py:101-128, evaluated on device; returns host arrays."""
    from .effective import pore_average_device

    _check_velocity(indicator, u)
    dev = require_cuda()
    t = torch()
    ud = to_device(u, dev, t.float64)
    if not bool(t.isfinite(ud).all()):
        raise ValueError("velocity field contains non-finite values")
    H = solid_on_device(indicator, dev).to(t.float64)
    pore = 1.0 - H
    try:
        u_bar = np.asarray(pore_average_device(ud, indicator, dev), dtype=float)
    except ValueError as exc:
        raise ValueError("cannot form the pore-averaged velocity: no pore cells") from exc
    g = np.asarray(cfg.composition_gradient, dtype=float)
    diff = pore + cfg.eta * H
    adv = cfg.pe * pore * ud
    forcing = cfg.pe * pore * float(u_bar @ g)
    nb = float(np.linalg.norm(u_bar))
    b0_vec = cfg.b0 * u_bar / nb if nb > 0.0 else np.zeros(indicator.grid.dim)
    return MediumCoefficients(diff.cpu().numpy(), adv.cpu().numpy(), forcing.cpu().numpy(), u_bar, b0_vec)


def _params(cfg: TransportConfig, max_iter: int) -> N.TransportParams:
    P = N.TransportParams()
    P.pe, P.eta, P.a0, P.b0, P.eps = cfg.pe, cfg.eta, cfg.a0, cfg.b0, cfg.eps
    P.composition_gradient = N.dbl_array(cfg.composition_gradient, 3)
    P.max_iter = int(max_iter)
    return P


class TransportSolver:
    """Device-resident comparison-medium driver (begin / iterate / end)."""

    def __init__(self, indicator, u_dev, cfg: TransportConfig, state: DeviceTransportState, device=None,
                 history_rows: int | None = None, pipeline: str | None = None, plan_slot: int = 0):
        self.device = require_cuda(device)
        self.indicator, self.cfg, self.state, self.u = indicator, cfg, state, u_dev
        self.plan = get_plan(indicator.grid.dims, cfg.symbol_mode, self.device, plan_slot)
        t = torch()
        self.rows = int(history_rows or cfg.max_iter)
        self.history = t.empty(self.rows * 4, dtype=t.float64, device=self.device)
        self.solid = solid_on_device(indicator, self.device)
        self.result = N.TransportResult()
        self._params = _params(cfg, min(cfg.max_iter, self.rows))
        self.pipeline_request = pipeline or os.environ.get("POREFLOW_B200_PIPELINE", "auto")
        if self.pipeline_request not in ("auto", "fused", "cufft"):
            raise ValueError("pipeline must be 'auto', 'fused' or 'cufft'")

    @property
    def pipeline(self) -> str:
        return {0: "cufft", 1: "fused"}.get(N.load().pf_transport_pipeline(self.plan.handle), "none")

    def begin(self):
        h = self.plan.bind_stream()
        N.check(N.load().pf_plan_set_fused(h, 0 if self.pipeline_request == "cufft" else 1))
        s = self.state
        N.check(N.load().pf_transport_begin(h, ctypes.byref(self._params), self.solid.data_ptr(), self.u.data_ptr(),
                                            s.chi.data_ptr(), s.grad_chi.data_ptr(), self.history.data_ptr(),
                                            ctypes.byref(self.result)))
        if self.pipeline_request == "fused" and self.pipeline != "fused":
            raise ValueError(f"fused pipeline unsupported for grid {self.indicator.grid.dims}")
        return self

    def iterate(self, n_iter: int, poll: bool = True):
        N.check(N.load().pf_transport_iterate(self.plan.handle, int(n_iter), 1 if poll else 0,
                                              ctypes.byref(self.result)))
        return self.result

    def end(self):
        N.check(N.load().pf_transport_end(self.plan.handle, ctypes.byref(self.result)))
        self.state.iterations = int(self.result.iterations)
        return self.result

    def report(self) -> ConvergenceReport:
        r = self.result
        it = int(r.iterations)
        hist = self.history[: it * 4].view(it, 4).cpu().numpy()
        d = self.indicator.grid.dim
        b0v = tuple(float(x) for x in r.b0_vec[:d])
        g = tuple(float(x) for x in np.asarray(self.cfg.composition_gradient, dtype=float))
        return ConvergenceReport(
            REPORT_COLUMNS, hist, converged=bool(r.converged), iterations=it, diverged=bool(r.diverged),
            reason=_REASONS[int(r.reason)],
            meta={"symbol_mode": self.cfg.symbol_mode, "eps": self.cfg.eps, "pe": self.cfg.pe,
                  "eta": self.cfg.eta, "a0": self.cfg.a0, "b0": self.cfg.b0, "b0_vec": b0v,
                  "composition_gradient": g, "pipeline": self.pipeline})


def solve_transport_device(indicator: IndicatorField, u, cfg: TransportConfig | None = None, init=None,
                           device=None, pipeline: str | None = None):
    """Device-resident ``solve_transport``: returns (DeviceTransportState, ConvergenceReport)."""
    cfg = cfg or TransportConfig()
    grid = indicator.grid
    if len(cfg.composition_gradient) != grid.dim:
        raise ValueError("composition_gradient dimension does not match the grid")
    _check_velocity(indicator, u)
    dev = require_cuda(device)
    t = torch()
    ud = to_device(u, dev, t.float64)
    if init is not None:
        good = tuple(init.chi.shape) == grid.dims and tuple(init.grad_chi.shape) == (grid.dim, *grid.dims)
        if not good:
            raise ValueError("warm-start state has wrong shape or non-finite values")
        chi = to_device(init.chi, dev, t.float64).clone()
        gch = to_device(init.grad_chi, dev, t.float64).clone()
        if not (bool(t.isfinite(chi).all()) and bool(t.isfinite(gch).all())):
            raise ValueError("warm-start state has wrong shape or non-finite values")
    else:
        chi = t.zeros(grid.dims, dtype=t.float64, device=dev)
        gch = t.zeros((grid.dim, *grid.dims), dtype=t.float64, device=dev)
    state = DeviceTransportState(chi, gch)
    solver = TransportSolver(indicator, ud, cfg, state, dev, pipeline=pipeline)
    solver.begin()
    solver.iterate(cfg.max_iter, poll=True)
    solver.end()
    return state, solver.report()


def solve_transport(indicator: IndicatorField, u, cfg: TransportConfig | None = None,
                    init: TransportState | None = None):
    """Drop-in for reference ``solve_transport`` (transport.py:180-268)."""
    state, report = solve_transport_device(indicator, u, cfg, init)
    return state.to_host(), report


# ---------------------------------------------------------------- step helpers
# (transport.py:131-177) on the device; numpy in -> numpy out, CUDA tensors stay.

def residual_rhs(state, coeffs: MediumCoefficients, cfg: TransportConfig, symbols):
    """Spectral right-hand side (transport.py:131-151): the polarization
    (pure.py:71-87) in real space, its transforms, then s_hat + sum_c 1j*kappa_c*w_hat[c]
    in the reference's accumulation order."""
    from . import _devops as D
    from .backends import cuda as K

    host = not any(D.is_tensor(x) for x in (state.grad_chi, coeffs.diffusivity))
    dev = D.device_of(state.grad_chi, coeffs.diffusivity)
    d = symbols.grid.dim
    w, s = K.transport_polarization(D.real(state.grad_chi, dev), D.real(coeffs.diffusivity, dev),
                                    D.real(coeffs.advection, dev), D.real(coeffs.forcing, dev), cfg.a0,
                                    np.asarray(coeffs.b0_vec, dtype=float),
                                    np.asarray(cfg.composition_gradient, dtype=float))
    w_hat = D.fftn_t(w, d)
    s_hat = D.fftn_t(s, d)
    return D.out_like(D.div_t(w_hat, D.kappa_tables(symbols, dev), d, base=s_hat), host)


def update_concentration(f_hat, cfg: TransportConfig, symbols, b0_vec):
    """Uniform-medium solve per mode (transport.py:154-177): returns (chi, grad_chi),
    the mode update (pure.py:90-115) with a zero flux part, then Re ifft of both."""
    from . import _devops as D
    from .backends import cuda as K

    host = not D.is_tensor(f_hat)
    dev = D.device_of(f_hat)
    t = torch()
    grid = symbols.grid
    F = D.cplx(f_hat, dev)
    w_hat = t.zeros((grid.dim, *grid.dims), dtype=t.complex128, device=dev)
    chi_hat, grad_hat = K.transport_mode_update(w_hat, F, D.kappa_tables(symbols, dev), D.real(symbols.lap, dev),
                                                cfg.a0, np.asarray(b0_vec, dtype=float))
    chi = D.ifftn_real_t(chi_hat, grid.dim)
    gch = D.ifftn_real_t(grad_hat, grid.dim)
    return D.out_like(chi, host), D.out_like(gch, host)
