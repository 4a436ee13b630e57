"""Independent solves run concurrently on one GPU.

The reference runs its unit solves one after another (cli.py:338-384) and runs
solver instances concurrently only on host threads (tests/test_backends.py:131-149).
Here each solve of a batch gets its own plan (``plan_slot``) and its own CUDA
stream, and the host hands every active solve a chunk of iterations (one graph
launch, no host synchronisation) before reading the solves' done flags.  Kernel
tails, the one-block finalize and the gated no-op passes of one solve then
overlap the other solves' passes: +15 % on 128^3 cells, +70 % on 64^3 cells.

Each solve's computation is exactly the sequential one (same kernels, same
reduction order), so a batch returns bit-for-bit the results of solving the
cells one by one (tests/test_gpu_batch.py).
"""

from __future__ import annotations

from typing import Sequence

from .device import require_cuda, solid_on_device, to_device, torch
from .grid import all_solid
from .stokes import DeviceAdmmState, PenaltyParams, StokesConfig, StokesSolver, _fast_path
from .transport import DeviceTransportState, TransportConfig, TransportSolver, _check_velocity


def _chunk(grid) -> int:
    n = 1
    for d in grid.dims:
        n *= int(d)
    return 4 if n >= (1 << 21) else (8 if n >= (1 << 15) else 16)


def _drive(jobs, chunk: int):
    """jobs: [(solver, stream)] already begun; iterate all to completion."""
    t = torch()
    active = list(jobs)
    while active:
        for s, st in active:
            with t.cuda.stream(st):
                s.iterate(chunk, poll=False)
        still = []
        for s, st in active:
            with t.cuda.stream(st):
                r = s.iterate(0, poll=True)  # reads this solve's control block (syncs its stream only)
            if not r.done:
                still.append((s, st))
        active = still


def solve_stokes_many_device(indicators: Sequence, cfgs: Sequence[StokesConfig],
                             penalties: PenaltyParams | Sequence[PenaltyParams] | None = None, device=None):
    """``solve_stokes_device`` for several (indicator, config) pairs at once, cold
    starts.  Returns [(DeviceAdmmState, ConvergenceReport)] in input order."""
    if len(indicators) != len(cfgs):
        raise ValueError("one StokesConfig per indicator")
    dev = require_cuda(device)
    t = torch()
    pens = list(penalties) if isinstance(penalties, (list, tuple)) else [penalties] * len(cfgs)
    out: list = [None] * len(cfgs)
    jobs, owners = [], []
    main = t.cuda.current_stream(dev)
    for k, (ind, cfg) in enumerate(zip(indicators, cfgs)):
        pen = pens[k] or PenaltyParams()
        grid = ind.grid
        if len(cfg.pressure_gradient) != grid.dim:
            raise ValueError("pressure_gradient dimension does not match the grid")
        if pen.b <= 0.0:
            raise ValueError("coupling penalty b must be positive for the zero mode")
        if all_solid(ind):
            out[k] = (DeviceAdmmState.zeros(grid, dev), _fast_path(grid, cfg, pen))
            continue
        st = t.cuda.Stream(dev)
        st.wait_stream(main)
        with t.cuda.stream(st):
            state = DeviceAdmmState.zeros(grid, dev)
            solver = StokesSolver(ind, cfg, pen, state, dev, plan_slot=k, cold=True).begin()
        jobs.append((solver, st))
        owners.append((k, state))
    if jobs:
        _drive(jobs, min(_chunk(ind.grid) for ind in indicators))
    for (solver, st), (k, state) in zip(jobs, owners):
        with t.cuda.stream(st):
            solver.end()
            out[k] = (state, solver.report())
        main.wait_stream(st)
    return out


def solve_transport_many_device(indicators: Sequence, velocities: Sequence, cfgs: Sequence[TransportConfig],
                                device=None):
    """``solve_transport_device`` for several (indicator, velocity, config)
    triples at once, cold starts.  Returns [(DeviceTransportState,
    ConvergenceReport)] in input order."""
    if not (len(indicators) == len(velocities) == len(cfgs)):
        raise ValueError("one velocity and one TransportConfig per indicator")
    dev = require_cuda(device)
    t = torch()
    out: list = [None] * len(cfgs)
    jobs, owners = [], []
    main = t.cuda.current_stream(dev)
    for k, (ind, u, cfg) in enumerate(zip(indicators, velocities, cfgs)):
        grid = ind.grid
        if len(cfg.composition_gradient) != grid.dim:
            raise ValueError("composition_gradient dimension does not match the grid")
        _check_velocity(ind, u)
        st = t.cuda.Stream(dev)
        st.wait_stream(main)
        with t.cuda.stream(st):
            ud = to_device(u, dev, t.float64)
            solid_on_device(ind, dev)
            state = DeviceTransportState(t.zeros(grid.dims, dtype=t.float64, device=dev),
                                         t.zeros((grid.dim, *grid.dims), dtype=t.float64, device=dev))
            solver = TransportSolver(ind, ud, cfg, state, dev, plan_slot=k).begin()
        jobs.append((solver, st))
        owners.append((k, state))
    if jobs:
        _drive(jobs, min(_chunk(ind.grid) for ind in indicators))
    for (solver, st), (k, state) in zip(jobs, owners):
        with t.cuda.stream(st):
            solver.end()
            out[k] = (state, solver.report())
        main.wait_stream(st)
    return out
