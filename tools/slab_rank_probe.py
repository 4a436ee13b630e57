"""Per-rank compute of a slab-decomposed cell whose full size does not fit one
GPU (BASELINE cfg 5, 1024^3): rank 0 of P run alone with the other ranks'
exchange blocks zero (tests/slab_loopback.py SoloComm), fused and cuFFT slab
pipelines, CUDA-event time per iteration.  Exchanges are local copies here, so
this is the rank's compute share; DESIGN.md §6 adds the NVLink exchange.

    python tools/slab_rank_probe.py [N] [P] [iters] [fused|both]
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_15554_b200 as pf  # noqa: E402
from paper_2312_15554_b200 import slab as S  # noqa: E402
from slab_loopback import SoloComm  # noqa: E402


def stage_times(sol, be, iters):
    """CUDA-event time of each fused-slab call (blocking exchange order)."""
    names = ("fused_pk", "fused_rs", "finalize", "fused_mf")
    ev = {k: [] for k in names}
    orig = {k: getattr(be, k) for k in names}

    def wrap(k):
        def f(*a, **kw):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = orig[k](*a, **kw)
            e1.record()
            ev[k].append((e0, e1))
            return r
        return f

    for k in names:
        setattr(be, k, wrap(k))
    sol.overlap = False
    sol.iterate(iters, poll=False)
    torch.cuda.synchronize()
    for k in names:
        setattr(be, k, orig[k])
    return {k: sum(a.elapsed_time(b) for a, b in v) / max(1, len(v)) for k, v in ev.items()}


def run(n, world, iters, fused, stages=False):
    dev = torch.device("cuda", 0)
    from paper_2312_15554_b200.grid import rasterize_packing_slab, random_sphere_packing

    lo, hi = S.slab_range(n, world, 0)
    solid_np = rasterize_packing_slab(random_sphere_packing(0), (n, n, n), lo, hi)  # rank 0's planes only
    cfg = pf.StokesConfig.with_tolerance(1e-12, pressure_gradient=(1.0, 0.0, 0.0), max_iter=iters + 8)
    be = S.DeviceSlabBackend((n, n, n), world, 0, "central", dev)
    be.bind()
    L = (hi - lo) * n * n
    st = {k: torch.zeros(3 * L, dtype=torch.float64, device=dev) for k in ("u", "u_tilde", "a", "lam")}
    st["q"] = torch.zeros(L, dtype=torch.float64, device=dev)
    solid = torch.as_tensor(solid_np).reshape(-1).to(dev)
    cls = S.FusedSlabStokes if fused else S.SlabStokes
    sol = cls(be, (n, n, n), cfg, pf.PenaltyParams(), solid, st, comm=SoloComm(world))
    sol.begin()
    sol.iterate(2, poll=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sol.iterate(iters, poll=False)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / iters
    st_ms = stage_times(sol, be, 3) if (stages and fused) else None
    sol.end()
    be.close()
    del sol, st, solid
    torch.cuda.empty_cache()
    return (ms, st_ms) if stages else ms


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    which = sys.argv[4] if len(sys.argv) > 4 else "both"
    res = {}
    for fused in ((True,) if which == "fused" else (True, False)):
        out = run(n, world, iters if fused else max(2, iters // 2), fused, stages=fused)
        ms, st = out if fused else (out, None)
        res["fused" if fused else "cufft"] = {"ms_per_iter": ms, "rank_voxel_iters_per_s": n ** 3 / world / (ms / 1e3)}
        if st:
            res["fused"]["stage_ms"] = st
    print(json.dumps({"grid": n, "ranks": world, "rank": 0, "pipelines": res}))
