"""First-call and steady-state cost of solve_stokes's state copy at 256^3 (20 iterations):
run once with the pinned-output path (default) and once with the staged ring
(POREFLOW_B200_PINNED_OUT_GB=0), each in a fresh process."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2312_15554_b200 as pf  # noqa: E402

n, it = 256, 20
bits = np.packbits(np.array(pf.random_packing_geometry(n, seed=0).values).ravel())
cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0, 0), max_iter=it)
torch.zeros(1, device="cuda")
for k in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    h, rep = pf.solve_stokes(pf.PackedIndicator(pf.UnitCellGrid((n, n, n)), bits), cfg)
    dt = time.perf_counter() - t
    print(f"call {k}: {dt * 1e3:.1f} ms", flush=True)
    del h
