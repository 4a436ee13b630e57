"""The product's slab driver (paper_2312_15554_b200/slab.py) over gloo with 1, 2
and 4 CPU ranks, the per-rank work done by a numpy test double: a
slab-decomposed solve reproduces the live-reference golden (same iteration
count, fields within 1e-10), so the exchange packing, global mode offsets,
all-reduced residual sums and lock-step stopping are right before the same
driver runs the pf_slab_* device work over NCCL."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run_rank(rank, world, port, case, q, overlap=True):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from slab_numpy_backend import NumpySlabBackend

        from paper_2312_15554_b200 import slab as S
        from paper_2312_15554_b200.stokes import PenaltyParams, StokesConfig

        z = np.load(os.path.join(HERE, "golden", f"{case}.npz"))
        solid = z["solid"]
        dims = solid.shape
        lo, hi = S.slab_range(dims[0], world, rank)
        pen = z["penalties"]
        penalties = PenaltyParams(alpha=float(pen[0]), beta=float(pen[1]), b=float(pen[2]), adaptive=bool(pen[3]))
        cfg = StokesConfig.with_tolerance(float(z["eps"]), pressure_gradient=tuple(z["g_p"]),
                                          max_iter=int(z["max_iter"]))
        be = NumpySlabBackend(dims, world, rank)
        L = (hi - lo) * dims[1] * dims[2]
        st = {k: torch.zeros(3 * L, dtype=torch.float64) for k in ("u", "u_tilde", "a", "lam")}
        st["q"] = torch.zeros(L, dtype=torch.float64)
        solid_t = torch.from_numpy(np.ascontiguousarray(solid[lo:hi], dtype=np.uint8)).reshape(-1)
        rep = S.SlabStokes(be, dims, cfg, penalties, solid_t, st, poll_every=4, overlap=overlap).solve()
        q.put((rank, lo, hi, {k: v.numpy().copy() for k, v in st.items()}, rep.iterations, rep.converged,
               rep.history))
    finally:
        if world > 1:
            dist.destroy_process_group()


def _solve(case, world, overlap=True):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_run_rank, args=(r, world, port, case, q, overlap)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


def _gather(res, dims):
    out = {}
    for k in ("u", "u_tilde", "a", "lam", "q"):
        parts = []
        for (_, lo, hi, st, *_r) in res:
            shp = (hi - lo, *dims[1:]) if k == "q" else (3, hi - lo, *dims[1:])
            parts.append(st[k].reshape(shp))
        out[k] = np.concatenate(parts, axis=0 if k == "q" else 1)
    return out


@pytest.mark.parametrize("case,world,overlap", [("stokes_sphere16_stiff", 1, True), ("stokes_sphere16_stiff", 4, True),
                                                ("stokes_random_trunc", 2, True), ("stokes_random_trunc", 2, False)])
def test_slab_driver_reproduces_reference(golden, case, world, overlap):
    """sphere16: stiff, converged (943 it); random_trunc: 10x12x9 (odd N2), adaptive, 40 it.
    overlap = the component-pipelined async exchanges (default), else blocking."""
    z = golden(case)
    res = _solve(case, world, overlap)
    its = {r[4] for r in res}
    assert its == {int(z["iterations"])}, its  # every rank stops at the reference's iteration
    for r in res:
        np.testing.assert_array_equal(r[6], res[0][6])  # identical histories on all ranks
    f = _gather(res, z["solid"].shape)
    for k, ref in (("u", z["u"]), ("u_tilde", z["u_tilde"]), ("a", z["a"]), ("lam", z["lam"]), ("q", z["q"])):
        err = np.linalg.norm(f[k] - ref) / max(np.linalg.norm(ref), 1e-300)
        assert err <= 1e-10, (k, err)
