"""BASELINE-config goldens (cfg 1 adaptive, cfg 2 transport at 128^3, cfg 3
truncated at 256^3) from the LIVE reference package, run in the build container:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_baseline.py [part ...]

Parts (each writes one ``.npz`` next to this script, so a long run can be
resumed part by part):

* ``cfg3``   — 256^3 random packing (seed 0, SURVEY §8d cfg 3; geometry from the
  product's host generator ``grid.random_packing_geometry``, whose sha256 is
  stored), reference-default adaptive penalties, eps = 1e-5, from zero,
  truncated at ``max_iter`` = 40 for e1 and 8 for e3 (``stokes.py:313-427``;
  the truncation is the reference's own ``max_iter`` exit).
* ``cfg2``   — 128^3 SC sphere array (r = 0.25): Stokes e1 with stiff penalties
  (converged; the cfg-2 velocity), then ``solve_transport`` under that u with
  the cfg-2 settings (Pe = 50, eta = 0.01, a0 = 0.55, b0 = 1, eps = 1e-5, g = e1;
  ``transport.py:180-268``) and a converging Pe = 10 case.
* ``cfg1a``  — 64^3 SC sphere array, three load cases with the reference's
  DEFAULT adaptive penalties (``stokes.py:287-310``), eps = 1e-5, plus K.

Fields are too large to commit at these sizes, so each fixture keeps full
histories, iteration counts, final penalties, norms / maxima, and the fields at
4096 fixed voxels (``default_rng(0)`` choice).  Library versions are stored.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import scipy

os.environ.setdefault("POREFLOW_BACKEND", "pure")
import poreflow as pf  # noqa: E402  (the reference; never imported by the product)
from poreflow.spectral import make_symbols  # noqa: E402

OUT = Path(__file__).resolve().parent
ROOT = OUT.parents[1]
sys.path.insert(0, str(ROOT))
from paper_2312_15554_b200 import grid as our_grid  # noqa: E402  (host-only numpy generator)

VERSIONS = json.dumps({
    "numpy": np.__version__, "scipy": scipy.__version__, "python": sys.version.split()[0],
    "poreflow": pf.__version__, "cpus": os.cpu_count(),
})


def stiff():
    return pf.PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False)


def save(name, **arrays):
    arrays["versions"] = np.asarray(VERSIONS)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrays.items()}, flush=True)


def sample_idx(size, k=4096):
    return np.random.default_rng(0).choice(size, size=k, replace=False)


def field_summary(prefix, x, idx):
    x = np.asarray(x)
    return {f"{prefix}_sample": x.ravel()[idx], f"{prefix}_norm": np.asarray(np.linalg.norm(x)),
            f"{prefix}_max": np.asarray(np.abs(x).max())}


def stokes_summary(st, rep, n):
    idx_v = sample_idx(3 * n ** 3)
    idx_s = sample_idx(n ** 3)
    out = {}
    for k in ("u", "u_tilde", "a", "lam"):
        out.update(field_summary(k, getattr(st, k), idx_v))
    out.update(field_summary("q", st.q, idx_s))
    out.update(history=rep.history, iterations=np.asarray(rep.iterations),
               converged=np.asarray(rep.converged),
               final_penalties=np.asarray(rep.meta.get("final_penalties")))
    return out


def unit(ax):
    g = [0.0, 0.0, 0.0]
    g[ax] = 1.0
    return tuple(g)


def part_cfg3():
    n = 256
    ours = our_grid.random_packing_geometry(n, seed=0)
    ind = pf.IndicatorField(pf.UnitCellGrid((n, n, n)), ours.values)
    sha = hashlib.sha256(np.ascontiguousarray(ours.values).tobytes()).hexdigest()
    for ax, k in ((0, 40), (2, 8)):
        t0 = time.time()
        cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=unit(ax), max_iter=k)
        st, rep = pf.solve_stokes(ind, cfg)
        wall = time.time() - t0
        print("cfg3 load case", ax, rep.iterations, f"{wall:.1f}s", rep.meta.get("final_penalties"), flush=True)
        save(f"stokes_packing256_e{ax + 1}_trunc", n=np.asarray(n), seed=np.asarray(0), ind_sha256=np.asarray(sha),
             g_p=np.asarray(unit(ax)), eps=np.asarray(1e-5), max_iter=np.asarray(k), wall_s=np.asarray(wall),
             **stokes_summary(st, rep, n))


def part_cfg2():
    n = 128
    ind = pf.make_model_geometry(pf.UnitCellGrid((n, n, n)), radius=0.25)
    t0 = time.time()
    st, rep = pf.solve_stokes(ind, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=unit(0)), stiff())
    wall = time.time() - t0
    print("cfg2 stokes", rep.iterations, rep.converged, f"{wall:.1f}s", flush=True)
    save("stokes_sphere128_stiff", n=np.asarray(n), g_p=np.asarray(unit(0)), eps=np.asarray(1e-5),
         penalties=np.asarray([1000.0, 1000.0, 1000.0, 0.0]), wall_s=np.asarray(wall), **stokes_summary(st, rep, n))
    idx_v = sample_idx(3 * n ** 3)
    idx_s = sample_idx(n ** 3)
    for tag, pe, a0 in (("pe50", 50.0, 0.55), ("pe10", 10.0, 0.55)):
        tcfg = pf.TransportConfig(pe=pe, eta=0.01, a0=a0, b0=1.0, eps=1e-5, composition_gradient=unit(0))
        t0 = time.time()
        ts, tr = pf.solve_transport(ind, st.u, tcfg)
        wall = time.time() - t0
        print("cfg2 transport", tag, tr.iterations, tr.converged, tr.diverged, tr.reason, f"{wall:.1f}s", flush=True)
        out = {}
        out.update(field_summary("chi", ts.chi, idx_s))
        out.update(field_summary("grad_chi", ts.grad_chi, idx_v))
        save(f"transport_sphere128_{tag}", n=np.asarray(n), g_chi=np.asarray(unit(0)),
             params=np.asarray([pe, 0.01, a0, 1.0, 1e-5]), max_iter=np.asarray(tcfg.max_iter),
             history=tr.history, iterations=np.asarray(tr.iterations), converged=np.asarray(tr.converged),
             diverged=np.asarray(tr.diverged), reason=np.asarray(str(tr.reason)),
             b0_vec=np.asarray(tr.meta["b0_vec"]),
             wall_s=np.asarray(wall), **out)


def part_cfg1a():
    n = 64
    ind = pf.make_model_geometry(pf.UnitCellGrid((n, n, n)), radius=0.25)
    us, summ = [], {}
    for ax in range(3):
        t0 = time.time()
        st, rep = pf.solve_stokes(ind, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=unit(ax)))
        wall = time.time() - t0
        print("cfg1 adaptive load case", ax, rep.iterations, rep.converged, f"{wall:.1f}s", flush=True)
        us.append(st.u)
        for k, v in stokes_summary(st, rep, n).items():
            summ.setdefault(k, []).append(v)
        summ.setdefault("wall_s", []).append(wall)
    K = pf.permeability(us, ind, make_symbols(ind.grid, "central"))
    hist = summ.pop("history")
    maxlen = max(h.shape[0] for h in hist)
    H = np.full((3, maxlen, 15), np.nan)
    for i, h in enumerate(hist):
        H[i, : h.shape[0]] = h
    save("stokes_sphere64_cfg1_adaptive", n=np.asarray(n), history=H, K=K, eps=np.asarray(1e-5),
         **{k: np.stack([np.asarray(x) for x in v]) for k, v in summ.items()})


PARTS = {"cfg3": part_cfg3, "cfg2": part_cfg2, "cfg1a": part_cfg1a}

if __name__ == "__main__":
    for p in sys.argv[1:] or list(PARTS):
        PARTS[p]()
