"""e2e at 256^3, 20 iterations: solve_stokes (velocity copy overlapping the end step)
against solve_stokes_device + to_host (every field copied after the end step)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2312_15554_b200 as pf  # noqa: E402

n, it = 256, 20
bits = np.packbits(np.array(pf.random_packing_geometry(n, seed=0).values).ravel())
cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0, 0), max_iter=it)


def old():
    st, rep = pf.solve_stokes_device(pf.PackedIndicator(pf.UnitCellGrid((n, n, n)), bits), cfg)
    return st.to_host(), rep


def new():
    return pf.solve_stokes(pf.PackedIndicator(pf.UnitCellGrid((n, n, n)), bits), cfg)


ref = None
for name, f in [("old", old), ("new", new)] * 4:
    torch.cuda.synchronize()
    t = time.perf_counter()
    h, rep = f()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    if ref is None:
        ref = h
    same = all(np.array_equal(getattr(h, k), getattr(ref, k)) for k in ("u", "u_tilde", "q", "a", "lam"))
    print(f"{name}: {dt * 1e3:.1f} ms  e2e {it * n ** 3 / dt / 1e9:.2f} Gvox-it/s  identical={same}", flush=True)
