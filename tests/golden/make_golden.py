"""Generate golden fixtures from the LIVE reference package (``poreflow``).

Run in the build container, where the read-only reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small ``.npz`` files next to this script.  They pin two things:
the CPU oracle (``oracle/poreflow_oracle.py``) against the reference itself
(``tests/test_oracle_golden.py``, CPU), and the CUDA path against the same
numbers on the GPU box (``tests/test_gpu_parity.py``), where the reference is
absent.  Seeds, configs and library versions are stored inside each file.
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import scipy

os.environ.setdefault("POREFLOW_BACKEND", "pure")
import poreflow as pf  # noqa: E402  (the reference; never imported by the product)
from poreflow.backends import pure  # noqa: E402
from poreflow.spectral import make_symbols  # noqa: E402

OUT = Path(__file__).resolve().parent
VERSIONS = json.dumps({
    "numpy": np.__version__, "scipy": scipy.__version__, "python": sys.version.split()[0],
    "poreflow": pf.__version__,
})


def stiff():
    return pf.PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False)


def save(name, **arrays):
    arrays["versions"] = np.asarray(VERSIONS)
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrays.items()})


def kernels(name, dims, seed):
    rng = np.random.default_rng(seed)
    grid = pf.UnitCellGrid(dims)
    d = grid.dim
    out = {}
    for mode in ("central", "exact"):
        sym = make_symbols(grid, mode)
        c = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)  # noqa: E731
        q_hat, a_hat, ut_hat = c(*dims), c(d, *dims), c(d, *dims)
        u, a, lam, ut = (rng.standard_normal((d, *dims)) for _ in range(4))
        solid = rng.integers(0, 2, dims).astype(np.uint8)
        grad_chi = rng.standard_normal((d, *dims))
        diffu = rng.uniform(0.01, 1.0, dims)
        adv = rng.standard_normal((d, *dims))
        forcing = rng.standard_normal(dims)
        w_hat, s_hat = c(d, *dims), c(*dims)
        g_p = rng.standard_normal(d)
        b0v = rng.standard_normal(d)
        g_chi = rng.standard_normal(d)
        H = solid.astype(float)
        uh = pure.stokes_velocity_update(q_hat, a_hat, ut_hat, sym.kappa, sym.lap, sym.kappa_sq,
                                         1.3, 2.7, 0.9, g_p)
        utn = pure.aux_velocity_update(u, a, lam, H, 3.0, 1.7)
        an, ln = pure.multiplier_update(a, lam, u, ut, H, 3.0, 1.7)
        w, s = pure.transport_polarization(grad_chi, diffu, adv, forcing, 0.55, b0v, g_chi)
        ch, gh = pure.transport_mode_update(w_hat, s_hat, sym.kappa, sym.lap, 0.55, b0v)
        for k, v in dict(q_hat=q_hat, a_hat=a_hat, ut_hat=ut_hat, u=u, a=a, lam=lam, ut=ut,
                         solid=solid, grad_chi=grad_chi, diffusivity=diffu, advection=adv,
                         forcing=forcing, w_hat=w_hat, s_hat=s_hat, g_p=g_p, b0_vec=b0v,
                         g_chi=g_chi, out_u_hat=uh, out_u_tilde=utn, out_a=an, out_lam=ln,
                         out_w=w, out_s=s, out_chi_hat=ch, out_grad_hat=gh).items():
            out[f"{mode}_{k}"] = v
    save(name, dims=np.asarray(dims), **out)


def stokes_case(name, indicator, g, eps, penalties, max_iter=10_000, **extra):
    cfg = pf.StokesConfig.with_tolerance(eps, pressure_gradient=tuple(g), max_iter=max_iter)
    st, rep = pf.solve_stokes(indicator, cfg, penalties)
    print(name, "iterations", rep.iterations, "converged", rep.converged)
    pen = penalties or pf.PenaltyParams()
    save(name, solid=indicator.values, g_p=np.asarray(g, float), eps=np.asarray(eps),
         max_iter=np.asarray(max_iter),
         penalties=np.asarray([pen.alpha, pen.beta, pen.b, float(pen.adaptive)]),
         u=st.u, u_tilde=st.u_tilde, q=st.q, a=st.a, lam=st.lam, history=rep.history,
         iterations=np.asarray(rep.iterations), converged=np.asarray(rep.converged),
         final_penalties=np.asarray(rep.meta.get("final_penalties", pen.as_tuple())), **extra)
    return st, rep


def main():
    # kernel-level vectors (test_backends.py analogue), 2D and odd-sized 3D
    kernels("kernels_2d", (12, 8), 17)
    kernels("kernels_3d", (6, 5, 8), 5)

    # symbol known answer (test_spectral.py:59-72) is analytic; store the tables
    g3 = pf.UnitCellGrid((8, 6, 5))
    for mode in ("central", "exact"):
        s = make_symbols(g3, mode)
        save(f"symbols_{mode}", dims=np.asarray(g3.dims), k0=s.kappa[0], k1=s.kappa[1],
             k2=s.kappa[2], lap=s.lap, kappa_sq=s.kappa_sq)

    # Stokes: the reference's own 2D backend-parity case (test_backends.py:109-128)
    disk = pf.make_model_geometry(pf.UnitCellGrid((16, 16)), radius=0.25)
    stokes_case("stokes_disk16_stiff", disk, (1.0, 0.0), 1e-5, stiff())
    # 3D sphere, BASELINE cfg-1 geometry at 16^3: stiff and default-adaptive
    sph = pf.make_model_geometry(pf.UnitCellGrid((16, 16, 16)), radius=0.25)
    st16, _ = stokes_case("stokes_sphere16_stiff", sph, (1.0, 0.0, 0.0), 1e-5, stiff())
    sph12 = pf.make_model_geometry(pf.UnitCellGrid((12, 12, 12)), radius=0.3)
    stokes_case("stokes_sphere12_adaptive", sph12, (0.0, 1.0, 0.0), 1e-4, None)
    # non-cubic, odd axis, truncated (max_iter) run with adaptation active
    rng = np.random.default_rng(3)
    blob = pf.IndicatorField(pf.UnitCellGrid((10, 12, 9)), (rng.random((10, 12, 9)) < 0.2).astype(np.uint8))
    stokes_case("stokes_random_trunc", blob, (0.3, -0.2, 1.0), 1e-6, None, max_iter=40)
    # all-solid fast path
    allsolid = pf.IndicatorField(pf.UnitCellGrid((6, 6, 6)), np.ones((6, 6, 6), np.uint8))
    stokes_case("stokes_allsolid", allsolid, (1.0, 0.0, 0.0), 1e-5, None)

    # transport under the sphere flow (cfg-2 settings).  With this u, Pe=50 and
    # a0=0.55 trip the reference's divergence guard after 60 iterations, so the
    # converging fixtures use Pe=10 (a0=0.55) and Pe=50 (a0=1.0).
    for tag, (pe, a0, gvec) in {"pe10": (10.0, 0.55, (1.0, 0.0, 0.0)),
                                "pe50": (50.0, 1.0, (0.0, 1.0, 0.0)),
                                "pe50_guard": (50.0, 0.55, (1.0, 0.0, 0.0))}.items():
        tcfg = pf.TransportConfig(pe=pe, eta=0.01, a0=a0, b0=1.0, eps=1e-5,
                                  composition_gradient=gvec)
        ts, tr = pf.solve_transport(sph, st16.u, tcfg)
        print("transport", tag, tr.iterations, tr.converged, tr.diverged)
        save(f"transport_sphere16_{tag}", solid=sph.values, u=st16.u, g_chi=np.asarray(gvec),
             params=np.asarray([pe, 0.01, a0, 1.0, 1e-5]), max_iter=np.asarray(10_000),
             chi=ts.chi, grad_chi=ts.grad_chi,
             history=tr.history, iterations=np.asarray(tr.iterations),
             converged=np.asarray(tr.converged), diverged=np.asarray(tr.diverged),
             b0_vec=np.asarray(tr.meta["b0_vec"]))
    # divergence guard: a0 far below the contrast boundary (test_acceptance a0 sweep)
    dcfg = pf.TransportConfig(pe=50.0, eta=0.01, a0=0.05, b0=1.0, eps=1e-8,
                              composition_gradient=(0.0, 0.0, 1.0), max_iter=2000)
    ds, dr = pf.solve_transport(sph, st16.u, dcfg)
    print("diverging transport", dr.iterations, dr.diverged, dr.reason)
    save("transport_sphere16_diverge", solid=sph.values, u=st16.u, g_chi=np.asarray([0, 0, 1.0]),
         params=np.asarray([50.0, 0.01, 0.05, 1.0, 1e-8]), max_iter=np.asarray(2000),
         chi=ds.chi, grad_chi=ds.grad_chi, history=dr.history,
         iterations=np.asarray(dr.iterations), b0_vec=np.asarray(dr.meta["b0_vec"]),
         converged=np.asarray(dr.converged), diverged=np.asarray(dr.diverged))

    # effective tensors on an 8^3 sphere: 3 unit flows + 3 transports
    s8 = pf.make_model_geometry(pf.UnitCellGrid((8, 8, 8)), radius=0.3)
    us = []
    for ax in range(3):
        g = [0.0] * 3
        g[ax] = 1.0
        st, rep = pf.solve_stokes(s8, pf.StokesConfig.with_tolerance(1e-6, pressure_gradient=tuple(g)), stiff())
        assert rep.converged
        us.append(st.u)
    K = pf.permeability(us, s8, make_symbols(s8.grid, "central"))
    chis = []
    for ax in range(3):
        g = [0.0] * 3
        g[ax] = 1.0
        ts, tr = pf.solve_transport(s8, us[0], pf.TransportConfig(pe=10.0, eps=1e-6, composition_gradient=tuple(g), max_iter=50_000))
        assert tr.converged
        chis.append((ts.chi, ts.grad_chi))
    D = pf.diffusivity(us, chis, s8, 10.0)
    ubar = np.stack([pf.pore_average(u, s8) for u in us])
    save("effective_sphere8", solid=s8.values, u=np.stack(us), chi=np.stack([c[0] for c in chis]),
         grad_chi=np.stack([c[1] for c in chis]), K=K, D=D, pe=np.asarray(10.0), u_bar=ubar,
         porosity=np.asarray(pf.porosity(s8)))


if __name__ == "__main__":
    main()
