"""Extended-domain Stokes solver on B200 — drop-in for reference
``poreflow.stokes`` (pkg/src/poreflow/stokes.py).

Same dataclasses, validation, fast path and report contract as the reference;
the ADMM loop (stokes.py:375-417) runs entirely on device behind
``pf_stokes_*`` (include/poreflow_b200.h): a CUDA-graph loop body with a
device-side done flag, history rows written on device and copied back once.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, replace

import numpy as np

from . import _native as N
from .device import get_plan, require_cuda, solid_on_device, to_device, to_host_many, torch
from .grid import IndicatorField, all_solid
from .report import ConvergenceReport
from .spectral import CENTRAL, SYMBOL_MODES

CONSTRAINT_NAMES = ("solid", "divergence", "coupling")  # stokes.py:36

REPORT_COLUMNS = (  # stokes.py:38-43
    "r_p1", "r_p1_tol", "r_d1", "r_d1_tol",
    "r_p2", "r_p2_tol", "r_d2", "r_d2_tol",
    "r_p3", "r_p3_tol", "r_d3", "r_d3_tol",
    "alpha", "beta", "b",
)


@dataclass
class PenaltyParams:
    """stokes.py:46-76."""

    alpha: float = 1.0
    beta: float = 1.0
    b: float = 1.0
    adaptive: bool = True
    growth: tuple = (1.1, 1.1, 1.1)
    ratio_threshold: tuple = (20.0, 10.0, 30.0)
    floor: tuple = (1e-3, 1e-3, 1e-3)

    def __post_init__(self):
        if min(self.alpha, self.beta, self.b) <= 0.0:
            raise ValueError("penalty coefficients must be positive")
        if any(g <= 1.0 for g in self.growth):
            raise ValueError("growth factors must exceed 1")
        if any(t <= 1.0 for t in self.ratio_threshold):
            raise ValueError("ratio thresholds must exceed 1")
        if any(f <= 0.0 for f in self.floor):
            raise ValueError("floors must be positive")

    def as_tuple(self):
        return (self.alpha, self.beta, self.b)


@dataclass
class StokesConfig:
    """stokes.py:79-111 (central symbols by default)."""

    nu: float = 1.0
    pressure_gradient: tuple = (1.0, 0.0)
    eps_abs: float = 1e-5
    eps_rel: float = 1e-5
    max_iter: int = 10_000
    symbol_mode: str = CENTRAL

    def __post_init__(self):
        if self.nu <= 0.0:
            raise ValueError("viscosity must be positive")
        if self.eps_abs <= 0.0 or self.eps_rel < 0.0:
            raise ValueError("tolerances must be positive (eps_rel may be zero)")
        if self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")
        if self.symbol_mode not in SYMBOL_MODES:
            raise ValueError(f"symbol_mode must be one of {SYMBOL_MODES}")

    @classmethod
    def with_tolerance(cls, eps: float, **kwargs) -> "StokesConfig":
        return cls(eps_abs=eps, eps_rel=eps, **kwargs)


@dataclass
class AdmmState:
    """Iterate bundle (host numpy arrays).  stokes.py:114-139."""

    u: np.ndarray
    u_tilde: np.ndarray
    q: np.ndarray
    a: np.ndarray
    lam: np.ndarray
    iterations: int = 0

    @classmethod
    def zeros(cls, grid) -> "AdmmState":
        return cls(u=grid.zeros_vector(), u_tilde=grid.zeros_vector(), q=grid.zeros_scalar(),
                   a=grid.zeros_vector(), lam=grid.zeros_vector())

    def copy(self) -> "AdmmState":
        return AdmmState(self.u.copy(), self.u_tilde.copy(), self.q.copy(), self.a.copy(),
                         self.lam.copy(), self.iterations)


@dataclass
class ResidualPair:
    """stokes.py:142-151."""

    primal: float
    primal_tol: float
    dual: float
    dual_tol: float

    @property
    def passed(self) -> bool:
        return self.primal <= self.primal_tol and self.dual <= self.dual_tol


def adapt_penalties(penalties: PenaltyParams, pairs) -> PenaltyParams:
    """Residual balancing (stokes.py:287-310).  The device finalize kernel runs
    the same branch order each iteration; this host copy serves API callers."""
    values = list(penalties.as_tuple())
    for k, pair in enumerate(pairs):
        r_p, r_d = pair.primal, pair.dual
        if r_p == 0.0 and r_d == 0.0:
            continue
        grow = math.inf if r_d == 0.0 else r_p / r_d
        shrink = math.inf if r_p == 0.0 else r_d / r_p
        if grow > penalties.ratio_threshold[k]:
            values[k] = penalties.growth[k] * values[k]
        elif shrink > penalties.ratio_threshold[k]:
            values[k] = max(values[k] / penalties.growth[k], penalties.floor[k])
    return replace(penalties, alpha=values[0], beta=values[1], b=values[2])


@dataclass
class DeviceAdmmState:
    """The same iterate bundle as CUDA tensors (device-resident pipelines)."""

    u: object
    u_tilde: object
    q: object
    a: object
    lam: object
    iterations: int = 0

    @classmethod
    def zeros(cls, grid, device) -> "DeviceAdmmState":
        t = torch()
        z = lambda *s: t.zeros(s, dtype=t.float64, device=device)  # noqa: E731
        d = grid.dim
        return cls(z(d, *grid.dims), z(d, *grid.dims), z(*grid.dims), z(d, *grid.dims), z(d, *grid.dims))

    @classmethod
    def from_host(cls, st: AdmmState, device) -> "DeviceAdmmState":
        f = lambda a: to_device(np.asarray(a, dtype=np.float64), device)  # noqa: E731
        return cls(f(st.u), f(st.u_tilde), f(st.q), f(st.a), f(st.lam), st.iterations)

    def to_host(self) -> AdmmState:
        u, ut, q, a, lam = to_host_many([x.detach() for x in (self.u, self.u_tilde, self.q, self.a, self.lam)])
        return AdmmState(u, ut, q, a, lam, self.iterations)


def _params(cfg: StokesConfig, pen: PenaltyParams, max_iter: int) -> N.StokesParams:
    P = N.StokesParams()
    P.nu = cfg.nu
    P.pressure_gradient = N.dbl_array(cfg.pressure_gradient, 3)
    P.eps_abs, P.eps_rel = cfg.eps_abs, cfg.eps_rel
    P.max_iter = int(max_iter)
    P.alpha, P.beta, P.b = pen.alpha, pen.beta, pen.b
    P.adaptive = 1 if pen.adaptive else 0
    P.growth = N.dbl_array(pen.growth, 3)
    P.ratio_threshold = N.dbl_array(pen.ratio_threshold, 3)
    P.floor = N.dbl_array(pen.floor, 3)
    return P


def _validate_init(init, grid):
    """stokes.py:355-361."""
    for name in ("u", "u_tilde", "a", "lam"):
        arr = getattr(init, name)
        if tuple(arr.shape) != (grid.dim, *grid.dims) or not _all_finite(arr):
            raise ValueError(f"warm-start field {name!r} has wrong shape or non-finite values")
    if tuple(init.q.shape) != grid.dims or not _all_finite(init.q):
        raise ValueError("warm-start field 'q' has wrong shape or non-finite values")


def _all_finite(arr) -> bool:
    t = torch()
    if isinstance(arr, t.Tensor):
        return bool(t.isfinite(arr).all())
    return bool(np.isfinite(arr).all())


def _fast_path(grid, cfg, penalties):
    """All-solid cell: one trivially converged record (stokes.py:336-353)."""
    n_vec, n_sca = grid.dim * grid.n_pts, grid.n_pts
    tv, ts = math.sqrt(n_vec) * cfg.eps_abs, math.sqrt(n_sca) * cfg.eps_abs
    record = [0.0, tv, 0.0, tv, 0.0, ts, 0.0, ts, 0.0, tv, 0.0, tv,
              penalties.alpha, penalties.beta, penalties.b]
    return ConvergenceReport(REPORT_COLUMNS, np.asarray([record]), converged=True, iterations=1,
                             meta={"fast_path": "all-solid geometry"})


class StokesSolver:
    """Device-resident ADMM driver (begin / iterate / end of the C ABI).

    ``state`` is a DeviceAdmmState that the solver updates in place.
    """

    def __init__(self, indicator: IndicatorField, cfg: StokesConfig, penalties: PenaltyParams,
                 state: DeviceAdmmState, device=None, history_rows: int | None = None,
                 pipeline: str | None = None, plan_slot: int = 0, compact: bool | None = None,
                 cold: bool = False):
        """``cold``: the caller created ``state`` as zeros (the reference's default
        initial state), so the setup may skip its transforms (pf_plan_set_cold_start)."""
        self.device = require_cuda(device)
        self.cold = bool(cold)
        self.indicator, self.cfg, self.penalties, self.state = indicator, cfg, penalties, state
        grid = indicator.grid
        self.plan = get_plan(grid.dims, cfg.symbol_mode, self.device, plan_slot)
        t = torch()
        self.rows = int(history_rows or cfg.max_iter)
        self.history = t.empty(self.rows * len(REPORT_COLUMNS), dtype=t.float64, device=self.device)
        self.solid = solid_on_device(indicator, self.device)
        self.result = N.StokesResult()
        self._params = _params(cfg, penalties, min(cfg.max_iter, self.rows))
        self._begun = False
        self.pipeline_request = pipeline or os.environ.get("POREFLOW_B200_PIPELINE", "auto")
        self.compact = (os.environ.get("POREFLOW_B200_COMPACT", "1") != "0") if compact is None else bool(compact)
        if self.pipeline_request not in ("auto", "fused", "cufft"):
            raise ValueError("pipeline must be 'auto', 'fused' or 'cufft'")

    @property
    def pipeline(self) -> str:
        """Pipeline the device chose: 'fused' / 'fused-compact' (power-of-two cubes) or 'cufft' /
        'cufft-compact' (other grids; '-compact' = solid-only multiplier storage)."""
        return {0: "cufft", 1: "fused", 2: "fused-compact", 3: "cufft-compact"}.get(
            N.load().pf_stokes_pipeline(self.plan.handle), "none")

    def begin(self):
        lib = N.load()
        s = self.state
        h = self.plan.bind_stream()
        N.check(lib.pf_plan_set_fused(h, 0 if self.pipeline_request == "cufft" else 1))
        N.check(lib.pf_plan_set_compact(h, 1 if self.compact else 0))
        N.check(lib.pf_plan_set_cold_start(h, 1 if self.cold else 0))
        N.check(lib.pf_stokes_begin(h, ctypes.byref(self._params), self.solid.data_ptr(), s.u.data_ptr(),
                                    s.u_tilde.data_ptr(), s.q.data_ptr(), s.a.data_ptr(), s.lam.data_ptr(),
                                    self.history.data_ptr()))
        self._begun = True
        if self.pipeline_request == "fused" and not self.pipeline.startswith("fused"):
            raise ValueError(f"fused pipeline unsupported for grid {self.indicator.grid.dims}")
        return self

    def iterate(self, n_iter: int, poll: bool = True):
        N.check(N.load().pf_stokes_iterate(self.plan.handle, int(n_iter), 1 if poll else 0,
                                           ctypes.byref(self.result)))
        return self.result

    def end(self):
        N.check(N.load().pf_stokes_end(self.plan.handle, ctypes.byref(self.result)))
        self._begun = False
        self.state.iterations = int(self.result.iterations)
        return self.result

    def report(self) -> ConvergenceReport:
        it = int(self.result.iterations)
        hist = self.history[: it * len(REPORT_COLUMNS)].view(it, len(REPORT_COLUMNS)).cpu().numpy()
        fp = tuple(float(x) for x in self.result.final_penalties)
        g_p = tuple(float(x) for x in self.cfg.pressure_gradient)
        return ConvergenceReport(
            REPORT_COLUMNS, hist, converged=bool(self.result.converged), iterations=it,
            meta={"symbol_mode": self.cfg.symbol_mode, "eps_abs": self.cfg.eps_abs,
                  "eps_rel": self.cfg.eps_rel, "nu": self.cfg.nu, "pressure_gradient": g_p,
                  "final_penalties": fp, "pipeline": self.pipeline})


def solve_stokes_device(indicator: IndicatorField, cfg: StokesConfig | None = None,
                        penalties: PenaltyParams | None = None, init=None, device=None,
                        pipeline: str | None = None, compact: bool | None = None):
    """Device-resident ``solve_stokes``: returns (DeviceAdmmState, ConvergenceReport)."""
    cfg = cfg or StokesConfig()
    penalties = penalties or PenaltyParams()
    grid = indicator.grid
    if len(cfg.pressure_gradient) != grid.dim:
        raise ValueError("pressure_gradient dimension does not match the grid")
    if penalties.b <= 0.0:
        raise ValueError("coupling penalty b must be positive for the zero mode")
    dev = require_cuda(device)
    if all_solid(indicator):
        return DeviceAdmmState.zeros(grid, dev), _fast_path(grid, cfg, penalties)
    if init is not None:
        _validate_init(init, grid)
        if isinstance(init, DeviceAdmmState):
            t = torch()
            c = lambda x: x.to(dev, t.float64).clone()  # noqa: E731
            state = DeviceAdmmState(c(init.u), c(init.u_tilde), c(init.q), c(init.a), c(init.lam))
        else:
            state = DeviceAdmmState.from_host(init, dev)
    else:
        state = DeviceAdmmState.zeros(grid, dev)
    solver = StokesSolver(indicator, cfg, penalties, state, dev, pipeline=pipeline, compact=compact,
                          cold=init is None)
    solver.begin()
    solver.iterate(cfg.max_iter, poll=True)
    solver.end()
    return state, solver.report()


def solve_stokes(indicator: IndicatorField, cfg: StokesConfig | None = None,
                 penalties: PenaltyParams | None = None, init: AdmmState | None = None):
    """Drop-in for reference ``solve_stokes`` (stokes.py:313-427): numpy in, numpy out."""
    state, report = solve_stokes_device(indicator, cfg, penalties, init)
    return state.to_host(), report


# ---------------------------------------------------------------- step helpers
# (stokes.py:158-244): one ADMM sub-step each, on the device.  The state may hold
# numpy arrays (results come back as fresh numpy arrays) or CUDA tensors (results
# stay on the device).  The solver loop does not use these (it runs the fused /
# cuFFT pipelines); they serve callers and tests written against the reference's
# step-level API.

def _step_io(*xs):
    from . import _devops as D

    host = not any(D.is_tensor(x) for x in xs)
    return D, host, D.device_of(*xs)


def _solid_f64(indicator, dev):
    from . import _devops as D

    return D.real(indicator.as_float(), dev)


def step1_velocity_solve(state, cfg: StokesConfig, penalties: PenaltyParams, symbols):
    """Velocity stationarity solve (stokes.py:158-180): the rank-one Green's
    operator on fft(q), fft(a), fft(u_tilde); returns Re ifft(u_hat)."""
    if penalties.b <= 0.0:
        raise ValueError("coupling penalty b must be positive for the zero mode")
    from .backends import cuda as K

    D, host, dev = _step_io(state.u, state.q, state.a, state.u_tilde)
    d = symbols.grid.dim
    q_hat = D.fftn_t(D.real(state.q, dev), d)
    a_hat = D.fftn_t(D.real(state.a, dev), d)
    ut_hat = D.fftn_t(D.real(state.u_tilde, dev), d)
    u_hat = K.stokes_velocity_update(q_hat, a_hat, ut_hat, D.kappa_tables(symbols, dev), D.real(symbols.lap, dev),
                                     D.real(symbols.kappa_sq, dev), cfg.nu, penalties.beta, penalties.b,
                                     np.asarray(cfg.pressure_gradient, dtype=float))
    return D.out_like(D.ifftn_real_t(u_hat, d), host)


def step2_aux_update(u, state, penalties: PenaltyParams, indicator: IndicatorField):
    """Pointwise auxiliary-velocity update (stokes.py:183-194, pure.py:59-61)."""
    from .backends import cuda as K

    D, host, dev = _step_io(u, state.a, state.lam)
    ut = K.aux_velocity_update(D.real(u, dev), D.real(state.a, dev), D.real(state.lam, dev),
                               _solid_f64(indicator, dev), penalties.alpha, penalties.b)
    return D.out_like(ut, host)


def _div_real(u_dev, symbols, dev):
    from . import _devops as D

    d = symbols.grid.dim
    return D.ifftn_real_t(D.div_t(D.fftn_t(u_dev, d), D.kappa_tables(symbols, dev), d), d)


def step3_multiplier_update(u, u_tilde, state, penalties: PenaltyParams, indicator: IndicatorField, symbols):
    """Multiplier ascent (stokes.py:197-220): returns (q, a, lam); q' = q - beta*div(u)
    with its mean projected out."""
    from .backends import cuda as K

    D, host, dev = _step_io(u, u_tilde, state.q, state.a, state.lam)
    U = D.real(u, dev)
    div_u = _div_real(U, symbols, dev)
    a_new, lam_new = K.multiplier_update(D.real(state.a, dev), D.real(state.lam, dev), U, D.real(u_tilde, dev),
                                         _solid_f64(indicator, dev), penalties.alpha, penalties.b)
    q_new = D.q_update_t(D.real(state.q, dev), div_u, penalties.beta)
    return D.out_like(q_new, host), D.out_like(a_new, host), D.out_like(lam_new, host)


def residuals_and_tolerances(state_prev, state_next, penalties: PenaltyParams, cfg: StokesConfig,
                             indicator: IndicatorField, symbols):
    """The three primal/dual residual pairs with their tolerances (stokes.py:223-284):
    divergences and the nine norms on the device, the pair arithmetic on the host
    exactly as ``_residual_pairs``."""
    D, _, dev = _step_io(state_prev.u, state_next.u)
    Un, Up = D.real(state_next.u, dev), D.real(state_prev.u, dev)
    UTn, UTp = D.real(state_next.u_tilde, dev), D.real(state_prev.u_tilde, dev)
    H = _solid_f64(indicator, dev)
    div_prev = _div_real(Up, symbols, dev)
    div_next = _div_real(Un, symbols, dev)
    n_vec = int(Un.numel())
    n_sca = int(np.prod(tuple(state_next.q.shape)))
    eps_abs, eps_rel = cfg.eps_abs, cfg.eps_rel

    r_p1 = D.norm_t(UTn, None, H)
    r_d1 = penalties.alpha * D.norm_t(UTn, UTp, H)
    lam_norm = D.norm_t(D.real(state_next.lam, dev))
    pair1 = ResidualPair(r_p1, math.sqrt(n_vec) * eps_abs + eps_rel * max(r_p1, lam_norm), r_d1,
                         math.sqrt(n_vec) * eps_abs + eps_rel * lam_norm)
    r_p2 = D.norm_t(div_next)
    r_d2 = penalties.beta * D.norm_t(div_next, div_prev)
    q_norm = D.norm_t(D.real(state_next.q, dev))
    pair2 = ResidualPair(r_p2, math.sqrt(n_sca) * eps_abs + eps_rel * max(r_p2, q_norm), r_d2,
                         math.sqrt(n_sca) * eps_abs + eps_rel * q_norm)
    r_p3 = D.norm_t(Un, UTn)
    r_d3 = penalties.b * D.norm_t(Un, Up)
    a_norm = D.norm_t(D.real(state_next.a, dev))
    pair3 = ResidualPair(r_p3, math.sqrt(n_vec) * eps_abs + eps_rel * max(r_p3, a_norm), r_d3,
                         math.sqrt(n_vec) * eps_abs + eps_rel * a_norm)
    return pair1, pair2, pair3
