"""Break the end-to-end solve_stokes time at 256^3 into its phases (bench e2e leg).

    python tools/e2e_probe.py [--iters 300]
"""
import argparse
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2312_15554_b200 as pf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--iters", type=int, default=300)
ap.add_argument("--packed", action="store_true", help="bit-packed indicator in (the bench e2e leg)")
a = ap.parse_args()
n = a.n
vals = np.array(pf.random_packing_geometry(n, seed=0).values)
mk = lambda it: pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0, 0), max_iter=it)  # noqa: E731
pf.solve_stokes(pf.IndicatorField(pf.UnitCellGrid((n, n, n)), vals), mk(5))  # warm: plan, staging, libs
torch.cuda.synchronize()
dev = torch.device("cuda", 0)
T = {}
t = time.perf_counter()
ind = (pf.PackedIndicator(pf.UnitCellGrid((n, n, n)), np.packbits(vals.ravel())) if a.packed
       else pf.IndicatorField(pf.UnitCellGrid((n, n, n)), vals))
T["indicator"] = time.perf_counter() - t
t = time.perf_counter()
st = pf.DeviceAdmmState.zeros(ind.grid, dev)
s = pf.StokesSolver(ind, mk(a.iters), pf.PenaltyParams(), st, dev)
torch.cuda.synchronize()
T["state+solver"] = time.perf_counter() - t
t = time.perf_counter()
s.begin()
torch.cuda.synchronize()
T["begin (H2D, setup)"] = time.perf_counter() - t
t = time.perf_counter()
s.iterate(a.iters, poll=True)
torch.cuda.synchronize()
T["iterate"] = time.perf_counter() - t
t = time.perf_counter()
s.end()
torch.cuda.synchronize()
T["end (teardown)"] = time.perf_counter() - t
t = time.perf_counter()
rep = s.report()
T["report"] = time.perf_counter() - t
t = time.perf_counter()
h = st.to_host()
T["to_host"] = time.perf_counter() - t
tot = sum(T.values())
for k, v in T.items():
    print(f"{k:22s} {v * 1e3:9.2f} ms")
print(f"total {tot * 1e3:.1f} ms; iterate-only {n ** 3 * a.iters / T['iterate'] / 1e9:.2f} Gvox-it/s; "
      f"e2e {n ** 3 * a.iters / tot / 1e9:.2f} Gvox-it/s; pipeline {s.pipeline}")
x = st.u
p = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
for _ in range(2):
    t = time.perf_counter()
    p.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"pinned D2H {x.numel() * 8 / dt / 1e9:.1f} GB/s")
t = time.perf_counter()
q = np.empty(x.shape)
q[...] = p.numpy()
print(f"pinned->numpy memcpy {x.numel() * 8 / (time.perf_counter() - t) / 1e9:.1f} GB/s")
