"""Run flow and outputs on the device solvers — the reference's ``cli.run``
(pkg/src/poreflow/cli.py:264-487) without its INI/argparse front end: geometry →
d unit-pressure-gradient Stokes solves → physical flow by superposition → d
unit-composition-gradient transport solves under it → K*, D* → ``report.json``
(schema ``poreflow-report/1``), residual-history CSVs and field files in the
reference's formats (``fieldio``).  Parameter sweeps (cli.py:417-462) are
independent solves and run through the ensemble executor, so under
``torch.distributed`` their entries shard across ranks.

Same report structure, keys and exit codes as the reference; the difference is
that every solve is device-resident (`*_device` solvers, fields never leave the
GPU until a field file asks for them) and geometry may be 3D (the reference's
run geometries and VTK export are 2D only).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from .batch import solve_stokes_many_device, solve_transport_many_device
from .device import require_cuda, to_host
from .effective import EffectiveTensors, diffusivity, permeability, pore_average_device
from .ensemble import CellJob, run_ensemble
from .fieldio import export_field, load_indicator_raster, write_history_csv, write_indicator, write_report_json
from .grid import IndicatorField, UnitCellGrid, make_model_geometry, porosity, random_packing_geometry
from .stokes import PenaltyParams, StokesConfig, solve_stokes_device
from .transport import TransportConfig, solve_transport_device

REPORT_SCHEMA = "poreflow-report/1"  # cli.py:39
EXIT_OK, EXIT_USAGE, EXIT_NOT_CONVERGED = 0, 1, 2  # cli.py:40-42
SWEEP_PARAMS = ("alpha", "beta", "b", "a0", "b0", "eta", "pe", "tol", "resolution")  # cli.py:45


class ConfigError(ValueError):
    pass


@dataclass
class GeometrySpec:
    """cli.py:51-73.  ``disk`` / ``raster`` as the reference; ``ball`` (the
    centred ball of ``make_model_geometry`` in ``dim`` dimensions) and
    ``packing`` (the 3D random sphere packing of SURVEY §8d) are new."""

    kind: str
    radius: float = 0.25
    resolution: int = 128
    path: str = ""
    threshold: float = 0.5
    dim: int = 3
    seed: int = 0

    def build(self) -> IndicatorField:
        if self.kind == "disk":
            return make_model_geometry(UnitCellGrid((self.resolution,) * 2), radius=self.radius)
        if self.kind == "ball":
            return make_model_geometry(UnitCellGrid((self.resolution,) * self.dim), radius=self.radius)
        if self.kind == "raster":
            return load_indicator_raster(self.path, self.threshold)
        if self.kind == "packing":
            return random_packing_geometry(self.resolution, seed=self.seed)
        raise ConfigError(f"unknown geometry kind {self.kind!r}")

    def describe(self) -> dict:
        if self.kind == "disk":
            return {"kind": "disk", "radius": self.radius, "resolution": self.resolution}
        if self.kind == "raster":
            return {"kind": "raster", "path": self.path, "threshold": self.threshold}
        if self.kind == "ball":
            return {"kind": "ball", "radius": self.radius, "resolution": self.resolution, "dim": self.dim}
        return {"kind": self.kind, "resolution": self.resolution, "seed": self.seed}


@dataclass
class OutputSpec:
    """cli.py:76-80."""

    out_dir: str = "."
    fields: tuple = ()
    formats: tuple = ("csv",)
    histories: bool = True


@dataclass
class SweepSpec:
    """cli.py:83-86."""

    param: str
    values: tuple

    def __post_init__(self):
        if self.param not in SWEEP_PARAMS:
            raise ConfigError(f"sweep parameter must be one of {SWEEP_PARAMS}")


@dataclass
class RunConfig:
    """cli.py:89-96."""

    geometry: GeometrySpec
    stokes: StokesConfig = field(default_factory=StokesConfig)
    transport: TransportConfig = field(default_factory=TransportConfig)
    penalties: PenaltyParams = field(default_factory=PenaltyParams)
    output: OutputSpec = field(default_factory=OutputSpec)
    sweep: SweepSpec | None = None


def _unit_vector(dim: int, axis: int) -> tuple:
    e = [0.0] * dim
    e[axis] = 1.0
    return tuple(e)


def solve_report(report) -> dict:
    """cli.py:270-279."""
    entry = {"converged": bool(report.converged), "diverged": bool(report.diverged),
             "iterations": int(report.iterations), "final": report.final()}
    if report.reason:
        entry["reason"] = report.reason
    return entry


def run(config: RunConfig, device=None) -> tuple[dict, int]:
    """Execute one configured run (cli.py:282-414); returns (report, exit code)."""
    dev = require_cuda(device)
    out_dir = Path(config.output.out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    from . import __version__

    timing: dict = {}
    report: dict = {
        "schema": REPORT_SCHEMA,
        "version": __version__,
        "config": {"geometry": config.geometry.describe(), "stokes": vars(config.stokes).copy(),
                   "transport": vars(config.transport).copy(), "penalties": vars(config.penalties).copy()},
    }
    t0 = time.perf_counter()
    indicator = config.geometry.build()
    grid = indicator.grid
    phi_p = porosity(indicator)
    timing["geometry_s"] = time.perf_counter() - t0
    report["geometry"] = {"dims": list(grid.dims), "porosity": phi_p, "n_pts": grid.n_pts}

    if config.sweep is not None:
        entries, ok = run_sweep(config, indicator, dev)
        report["sweep"] = {"param": config.sweep.param, "entries": entries}
        timing["total_s"] = time.perf_counter() - t0
        report["timing"] = timing
        _write_outputs(report, None, None, indicator, config, out_dir, histories=())
        return report, EXIT_OK if ok else EXIT_NOT_CONVERGED

    if phi_p == 0.0:  # cli.py:321-336
        report["flow"] = {"unit_solves": [], "note": "all-solid geometry: zero flow"}
        report["transport"] = {"skipped": "no pore cells: pore averages undefined"}
        report["effective"] = {"permeability": np.zeros((grid.dim, grid.dim)), "porosity": phi_p}
        timing["total_s"] = time.perf_counter() - t0
        report["timing"] = timing
        _write_outputs(report, None, None, indicator, config, out_dir, histories=())
        return report, EXIT_OK

    # flow: one unit solve per axis; the configured-direction flow by linearity (cli.py:338-359)
    t0_flow = time.perf_counter()
    unit_u, flow_entries, histories = [], [], []
    all_ok = True
    cfgs = [replace(config.stokes, pressure_gradient=_unit_vector(grid.dim, axis)) for axis in range(grid.dim)]
    # the unit solves are independent: concurrent on one GPU (batch.py), same results
    for axis, (state, conv) in enumerate(solve_stokes_many_device([indicator] * grid.dim, cfgs, config.penalties,
                                                                  dev)):
        unit_u.append(state.u)
        entry = solve_report(conv)
        entry["pressure_gradient"] = list(cfgs[axis].pressure_gradient)
        flow_entries.append(entry)
        histories.append((f"flow_history_axis{axis + 1}.csv", conv))
        all_ok &= conv.converged
    g_p = np.asarray(config.stokes.pressure_gradient, dtype=float)
    u_phys = sum(float(g_p[i]) * unit_u[i] for i in range(grid.dim))
    timing["flow_s"] = time.perf_counter() - t0_flow
    report["flow"] = {"symbol_mode": config.stokes.symbol_mode, "nu": config.stokes.nu,
                      "pressure_gradient": g_p.tolist(), "unit_solves": flow_entries,
                      "u_bar_physical": pore_average_device(u_phys, indicator, dev)}

    # transport: one unit solve per axis under the physical flow (cli.py:361-384)
    t0_tra = time.perf_counter()
    chis, tra_entries = [], []
    tcfgs = [replace(config.transport, composition_gradient=_unit_vector(grid.dim, axis)) for axis in range(grid.dim)]
    for axis, (t_state, t_conv) in enumerate(solve_transport_many_device([indicator] * grid.dim,
                                                                         [u_phys] * grid.dim, tcfgs, dev)):
        chis.append((t_state.chi, t_state.grad_chi))
        entry = solve_report(t_conv)
        entry["composition_gradient"] = list(tcfgs[axis].composition_gradient)
        tra_entries.append(entry)
        histories.append((f"transport_history_axis{axis + 1}.csv", t_conv))
        all_ok &= t_conv.converged
    g_chi = np.asarray(config.transport.composition_gradient, dtype=float)
    chi_phys = sum(float(g_chi[j]) * chis[j][0] for j in range(grid.dim))
    timing["transport_s"] = time.perf_counter() - t0_tra
    report["transport"] = {"symbol_mode": config.transport.symbol_mode, "pe": config.transport.pe,
                           "eta": config.transport.eta, "a0": config.transport.a0, "b0": config.transport.b0,
                           "composition_gradient": g_chi.tolist(), "unit_solves": tra_entries}

    # effective tensors from the unit solutions (cli.py:386-408)
    tensors = EffectiveTensors(
        permeability=permeability(unit_u, indicator, config.stokes.symbol_mode),
        diffusivity=diffusivity(unit_u, chis, indicator, config.transport.pe),
        porosity=phi_p,
        u_bar=np.stack([np.atleast_1d(pore_average_device(u, indicator, dev)) for u in unit_u]),
        meta={"nu": config.stokes.nu, "flow_tolerance": [config.stokes.eps_abs, config.stokes.eps_rel],
              "transport_tolerance": config.transport.eps, "flow_symbol_mode": config.stokes.symbol_mode,
              "transport_symbol_mode": config.transport.symbol_mode,
              "flow_iterations": [e["iterations"] for e in flow_entries],
              "transport_iterations": [e["iterations"] for e in tra_entries],
              "velocity_convention": "concentration solved under the configured-"
                                     "direction flow; unit flows enter the tensor"})
    report["effective"] = vars(tensors).copy()
    timing["total_s"] = time.perf_counter() - t0
    report["timing"] = timing
    _write_outputs(report, u_phys, chi_phys, indicator, config, out_dir, histories)
    return report, EXIT_OK if all_ok else EXIT_NOT_CONVERGED


def run_sweep(config: RunConfig, indicator: IndicatorField, device=None) -> tuple[list, bool]:
    """Re-run the affected stage per sweep value (cli.py:417-462).  Each value is
    an independent job of the ensemble executor: with an initialised process
    group the values shard across ranks and every rank returns all entries."""
    dev = require_cuda(device)
    param = config.sweep.param
    stokes_params, transport_params = {"alpha", "beta", "b"}, {"a0", "b0", "eta", "pe"}
    flow_cache: dict = {}

    def flow():
        # the flow does not depend on the transport parameters: solve it once per rank
        if "u" not in flow_cache:
            state, conv = solve_stokes_device(indicator, config.stokes, config.penalties, device=dev)
            flow_cache["u"], flow_cache["ok"] = state.u, conv.converged
        return flow_cache["u"]

    def solve(job: CellJob) -> dict:
        value = job.meta["value"]
        entry: dict = {"value": value}
        ok = True
        if param in stokes_params:
            pen = replace(config.penalties, **{param: value}, adaptive=False)
            _, conv = solve_stokes_device(indicator, config.stokes, pen, device=dev)
            entry["stokes"] = solve_report(conv)
            ok = conv.converged
        elif param in transport_params:
            cfg = replace(config.transport, **{param: value})
            _, conv = solve_transport_device(indicator, flow(), cfg, device=dev)
            entry["transport"] = solve_report(conv)
            ok = conv.converged and flow_cache["ok"]
        else:
            if param == "tol":
                ind = indicator
                sto = replace(config.stokes, eps_abs=value, eps_rel=value)
                tra = replace(config.transport, eps=value)
            else:  # resolution
                ind = replace(config.geometry, resolution=int(value)).build()
                sto, tra = config.stokes, config.transport
            state, conv_s = solve_stokes_device(ind, sto, config.penalties, device=dev)
            _, conv_t = solve_transport_device(ind, state.u, tra, device=dev)
            entry["stokes"] = solve_report(conv_s)
            entry["transport"] = solve_report(conv_t)
            ok = conv_s.converged and conv_t.converged
        return {"entry": entry, "ok": bool(ok)}

    n = int(np.prod(indicator.grid.dims))
    jobs = [CellJob(key=i, indicator=indicator, cost=float(n) * (v if param == "resolution" else 1.0),
                    meta={"value": v}) for i, v in enumerate(config.sweep.values)]
    results = run_ensemble(jobs, solve)
    entries = [results[i]["entry"] for i in range(len(jobs))]
    all_ok = all(results[i]["ok"] for i in range(len(jobs)))
    if param in transport_params and "ok" not in flow_cache:
        # ranks that drew no transport job still owe the reference's flow-convergence term
        flow()
    if param in transport_params:
        all_ok = all_ok and flow_cache["ok"]
    return entries, all_ok


def _write_outputs(report, u_phys, chi_phys, indicator, config, out_dir, histories):
    """History CSVs, requested fields and report.json (cli.py:465-487).  Field
    formats: ``csv`` (2D, as the reference), ``vtk`` (2D as the reference, 3D
    new), ``npy`` (new)."""
    written = []
    grid = indicator.grid
    for name, conv in histories:
        if config.output.histories:
            written.append(str(write_history_csv(conv, out_dir / name)))
    field_data = {"velocity": (u_phys, "velocity"), "concentration": (chi_phys, "concentration")}
    for name in config.output.fields:
        if name == "indicator":
            written.append(str(write_indicator(indicator, out_dir / ("indicator.csv" if grid.dim == 2
                                                                     else "indicator.npy"))))
            continue
        data, label = field_data.get(name, (None, name))
        if data is None:
            continue
        host = to_host(data) if hasattr(data, "device") else np.asarray(data)
        for fmt in config.output.formats:
            suffix = {"csv": ".csv", "vtk": ".vtk", "npy": ".npy"}.get(fmt, "." + fmt)
            paths = export_field(host, grid, fmt, out_dir / f"{label}{suffix}", label)
            written.extend(str(p) for p in paths)
    report["outputs"] = {"directory": str(out_dir), "files": sorted(written)}
    write_report_json(report, out_dir / "report.json")
