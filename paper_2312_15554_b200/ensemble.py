"""Ensembles of independent unit cells across GPUs (BASELINE cfgs 3-4).

Every (cell, load case) solve is independent, so the multi-GPU path is pure
sharding: one process per GPU (torchrun), a deterministic work-balanced
assignment of cells to ranks, no data-path collective, and one small
``all_gather_object`` of the per-cell results (tensors, iteration counts) at the
end.  The reference has no counterpart (it runs solver instances concurrently
only on host threads, tests/test_backends.py:131-149).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np


@dataclass
class CellJob:
    """One unit cell of an ensemble; ``cost`` orders the greedy assignment."""

    key: object
    indicator: object
    cost: float = 0.0
    meta: dict = field(default_factory=dict)


def default_cost(indicator, expected_iterations: float = 1.0) -> float:
    """Work estimate: voxels x expected iterations (per-iteration cost is linear in n)."""
    return float(np.prod(indicator.grid.dims)) * float(expected_iterations)


def shard(jobs: Sequence[CellJob], world: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of job indices to ``world`` ranks.

    Deterministic: jobs sorted by (-cost, index); ties between ranks go to the
    lowest rank.  Every job lands on exactly one rank.
    """
    if world < 1:
        raise ValueError("world size must be positive")
    order = sorted(range(len(jobs)), key=lambda i: (-float(jobs[i].cost), i))
    load = [0.0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += float(jobs[i].cost)
    for lst in out:
        lst.sort()
    return out


def run_ensemble(jobs: Sequence[CellJob], solve_fn: Callable[[CellJob], dict], group=None) -> dict:
    """Run this rank's shard with ``solve_fn`` and gather all results on every rank.

    Returns {job.key: result}.  Without an initialised process group it runs
    every job locally (world size 1).
    """
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    else:
        world, rank = 1, 0
    mine = shard(jobs, world)[rank]
    local = {jobs[i].key: solve_fn(jobs[i]) for i in mine}
    if world == 1:
        return local
    gathered: list = [None] * world
    dist.all_gather_object(gathered, local, group=group)
    out: dict = {}
    for part in gathered:
        out.update(part)
    return out


def permeability_job(cfg_kwargs=None, penalties=None, device=None):
    """A ``solve_fn`` computing the full permeability tensor of a 3D cell on this
    rank's GPU: d unit-pressure-gradient solves + ``permeability`` (cli.py:338-388
    flow, device-resident)."""

    def solve(job: CellJob) -> dict:
        from . import effective, stokes

        from .batch import solve_stokes_many_device

        ind = job.indicator
        d = ind.grid.dim
        cfgs = []
        for ax in range(d):
            g = [0.0] * d
            g[ax] = 1.0
            kw = dict(cfg_kwargs or {})
            eps = kw.pop("eps", 1e-5)
            cfgs.append(stokes.StokesConfig.with_tolerance(eps, pressure_gradient=tuple(g), **kw))
        res = solve_stokes_many_device([ind] * d, cfgs, penalties, device)  # the d load cases concurrently
        us = [st.u for st, _ in res]
        iters = [rep.iterations for _, rep in res]
        conv = [rep.converged for _, rep in res]
        # the CLI builds K's symbols from the Stokes symbol mode (cli.py:386-388)
        K = effective.permeability(us, ind, cfgs[0].symbol_mode)
        return {"K": K, "iterations": iters, "converged": conv}

    return solve
