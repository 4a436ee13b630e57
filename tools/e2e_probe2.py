"""Finer breakdown of the e2e fixed costs at 256^3 (state allocation, solver init,
begin/setup, teardown, copy-back), each phase bracketed by device syncs."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_2312_15554_b200 as pf  # noqa: E402

n = 256
vals = np.array(pf.random_packing_geometry(n, seed=0).values)
bits = np.packbits(vals.ravel())
mk = lambda it: pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0, 0), max_iter=it)  # noqa: E731
for rep in range(3):
    T = {}
    torch.cuda.synchronize()
    t = time.perf_counter()
    ind = pf.PackedIndicator(pf.UnitCellGrid((n, n, n)), bits)
    T["indicator"] = time.perf_counter() - t
    dev = torch.device("cuda", 0)
    t = time.perf_counter()
    st = pf.DeviceAdmmState.zeros(ind.grid, dev)
    torch.cuda.synchronize()
    T["zeros"] = time.perf_counter() - t
    t = time.perf_counter()
    s = pf.StokesSolver(ind, mk(20), pf.PenaltyParams(), st, dev, cold=True)
    torch.cuda.synchronize()
    T["solver_init"] = time.perf_counter() - t
    t = time.perf_counter()
    s.begin()
    torch.cuda.synchronize()
    T["begin"] = time.perf_counter() - t
    t = time.perf_counter()
    s.iterate(20, poll=True)
    torch.cuda.synchronize()
    T["iterate"] = time.perf_counter() - t
    t = time.perf_counter()
    s.end()
    torch.cuda.synchronize()
    T["end"] = time.perf_counter() - t
    t = time.perf_counter()
    s.report()
    h = st.to_host()
    T["report+to_host"] = time.perf_counter() - t
    print(rep, " ".join(f"{k} {v * 1e3:.2f}" for k, v in T.items()), f"total {sum(T.values()) * 1e3:.1f} ms")
