"""solve_stokes at 256^3 (20 iterations) called repeatedly: keeping every result
(three load cases, as cli.run does for K) and dropping each before the next (the
bench's pattern); per-call wall time."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2312_15554_b200 as pf  # noqa: E402

n, it = 256, 20
bits = np.packbits(np.array(pf.random_packing_geometry(n, seed=0).values).ravel())
ind = pf.PackedIndicator(pf.UnitCellGrid((n, n, n)), bits)
torch.zeros(1, device="cuda")
keep = []
for k in range(3):
    g = [0.0, 0.0, 0.0]
    g[k] = 1.0
    t = time.perf_counter()
    keep.append(pf.solve_stokes(ind, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=tuple(g), max_iter=it)))
    print(f"keep  call {k}: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
ref = keep[0][0].u.copy()
del keep
for k in range(4):
    t = time.perf_counter()
    st, rep = pf.solve_stokes(ind, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0, 0), max_iter=it))
    print(f"drop  call {k}: {(time.perf_counter() - t) * 1e3:.1f} ms  same={np.array_equal(st.u, ref)}", flush=True)
    del st
