"""BASELINE cfg-1 golden (64^3 simple-cubic sphere array, r = 0.25) from the LIVE
reference: three unit-pressure-gradient Stokes solves with stiff penalties at
eps = 1e-5, the permeability tensor K (Stokes symbols, cli.py:386-388), and
u sampled at 4096 fixed voxels per load case (the full fields are 6 MiB each).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cfg1.py
"""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import scipy

os.environ.setdefault("POREFLOW_BACKEND", "pure")
import poreflow as pf  # noqa: E402  (the reference)
from poreflow.spectral import make_symbols  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    n = 64
    ind = pf.make_model_geometry(pf.UnitCellGrid((n, n, n)), radius=0.25)
    pen = pf.PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False)
    rng = np.random.default_rng(0)
    sample = rng.choice(3 * n ** 3, size=4096, replace=False)
    us, its, hists, walls = [], [], [], []
    for ax in range(3):
        g = [0.0] * 3
        g[ax] = 1.0
        t0 = time.time()
        st, rep = pf.solve_stokes(ind, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=tuple(g)), pen)
        walls.append(time.time() - t0)
        print("load case", ax, rep.iterations, rep.converged, f"{walls[-1]:.1f}s", flush=True)
        us.append(st.u)
        its.append(rep.iterations)
        hists.append(rep.history)
    K = pf.permeability(us, ind, make_symbols(ind.grid, "central"))
    maxlen = max(h.shape[0] for h in hists)
    H = np.full((3, maxlen, 15), np.nan)
    for i, h in enumerate(hists):
        H[i, : h.shape[0]] = h
    np.savez_compressed(
        OUT / "stokes_sphere64_cfg1.npz", solid_packed=np.packbits(ind.values), dims=np.asarray([n, n, n]),
        iterations=np.asarray(its), history=H, K=K, sample=sample,
        u_sample=np.stack([u.ravel()[sample] for u in us]),
        u_norm=np.asarray([np.linalg.norm(u) for u in us]), u_max=np.asarray([np.abs(u).max() for u in us]),
        wall_s=np.asarray(walls),
        versions=np.asarray(json.dumps({"numpy": np.__version__, "scipy": scipy.__version__,
                                        "python": sys.version.split()[0], "cpus": os.cpu_count()})))
    print("K", K)


if __name__ == "__main__":
    main()
