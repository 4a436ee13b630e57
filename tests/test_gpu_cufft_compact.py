"""Solid-only multiplier storage on the general-grid (cuFFT) pipeline
(csrc/pf_stokes.cu k_stokes_local_c / k_form_r_fix_c / k_gcompact_move): the
same results as the full-storage path and the oracle, eligibility fallbacks
(a != 0 on a pore voxel, voxel counts that are not a multiple of 64), 2D grids."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELD_TOL = 1e-10


@pytest.fixture(scope="module")
def pf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_15554_b200 as pf

    return pf


def rel_l2(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def _hist_close(mine, ref, **kw):
    from parity_util import hist_close

    hist_close(mine, ref, kind="stokes", **kw)


@pytest.mark.parametrize("n", [40, 100])
def test_compact_matches_full_storage(pf, n):
    """The default adaptive penalties through b changes (asserted): solid-only storage
    against the full-storage cuFFT path on the same cell — same iterations and
    penalties, fields to round-off (pore voxels take u~' = u', a' = 0 exactly instead
    of through the division, an ulp-level difference)."""
    ind = pf.random_packing_geometry(n, seed=2)
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(0.0, 1.0, 0.0), max_iter=30)
    a, ra = pf.solve_stokes_device(ind, cfg, pipeline="cufft", compact=True)
    b, rb = pf.solve_stokes_device(ind, cfg, pipeline="cufft", compact=False)
    assert ra.meta["pipeline"] == "cufft-compact" and rb.meta["pipeline"] == "cufft"
    assert np.unique(ra.history[:-1, 14]).size > 1
    assert ra.iterations == rb.iterations == 30
    ha, hb = a.to_host(), b.to_host()
    for k in ("u", "u_tilde", "q", "a", "lam"):
        assert rel_l2(getattr(ha, k), getattr(hb, k)) <= 1e-12, k
    pore = np.asarray(ind.values) == 0
    assert (ha.a[:, pore] == 0.0).all()
    assert (ha.u_tilde[:, pore] == ha.u[:, pore]).all()
    _hist_close(ra.history, rb.history)
    np.testing.assert_allclose(ra.meta["final_penalties"], rb.meta["final_penalties"], rtol=1e-12)


def test_compact_warm_start_vs_oracle(pf):
    """Warm start from a state this path produced (a = 0 on pore voxels: eligible),
    with a nonzero pore lam (constant there: its |lam|^2 enters the finalize as a
    constant), against the oracle from the same state."""
    from oracle import poreflow_oracle as O

    n = 40
    ind = pf.random_packing_geometry(n, seed=3)
    g = (1.0, 0.0, 0.0)
    st0, _ = pf.solve_stokes(ind, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=g, max_iter=10))
    lam = st0.lam.copy()
    pore = np.asarray(ind.values) == 0
    lam[:, pore] = 0.01
    init = pf.AdmmState(st0.u, st0.u_tilde, st0.q, st0.a, lam)
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=g, max_iter=12)
    st, rep = pf.solve_stokes_device(ind, cfg, init=init, pipeline="cufft")
    assert rep.meta["pipeline"] == "cufft-compact"
    ost, ohist, _, oit, _ = O.solve_stokes(ind.values, g, 1e-5, 1e-5, max_iter=12,
                                           init=dict(u=st0.u, u_tilde=st0.u_tilde, q=st0.q, a=st0.a, lam=lam))
    assert rep.iterations == oit
    h = st.to_host()
    for k in ("u", "u_tilde", "q", "a", "lam"):
        assert rel_l2(getattr(h, k), ost[k]) <= FIELD_TOL, k
    assert (h.lam[:, pore] == 0.01).all()
    _hist_close(rep.history, ohist)


def test_compact_fallbacks(pf):
    """Full storage when a != 0 on some pore voxel, and when the voxel count is not a
    multiple of 64; both still match the oracle."""
    from oracle import poreflow_oracle as O

    ind = pf.random_packing_geometry(40, seed=3)
    g = (1.0, 0.0, 0.0)
    st0, _ = pf.solve_stokes(ind, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=g, max_iter=5))
    a = st0.a.copy()
    a[0, np.asarray(ind.values) == 0] = 1e-3
    init = pf.AdmmState(st0.u, st0.u_tilde, st0.q, a, st0.lam)
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=g, max_iter=6)
    st, rep = pf.solve_stokes_device(ind, cfg, init=init, pipeline="cufft")
    assert rep.meta["pipeline"] == "cufft"
    ost, _, _, oit, _ = O.solve_stokes(ind.values, g, 1e-5, 1e-5, max_iter=6,
                                       init=dict(u=st0.u, u_tilde=st0.u_tilde, q=st0.q, a=a, lam=st0.lam))
    assert rep.iterations == oit
    assert rel_l2(st.to_host().a, ost["a"]) <= FIELD_TOL

    odd = pf.random_packing_geometry(33, seed=1)  # 33^3 = 35937 voxels
    st, rep = pf.solve_stokes(odd, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=g, max_iter=8))
    assert rep.meta["pipeline"] == "cufft"
    ost, _, _, oit, _ = O.solve_stokes(odd.values, (1.0, 0.0, 0.0), 1e-5, 1e-5, max_iter=8)
    assert rep.iterations == oit and rel_l2(st.u, ost["u"]) <= FIELD_TOL


def test_compact_2d_vs_oracle(pf):
    """2D cell (D = 2 components), 48 x 32 = 1536 voxels: solid-only storage against the oracle."""
    from oracle import poreflow_oracle as O

    grid = pf.UnitCellGrid((48, 32))
    ind = pf.make_model_geometry(grid, radius=0.3)
    cfg = pf.StokesConfig.with_tolerance(1e-6, pressure_gradient=(1.0, 0.0), max_iter=200)
    st, rep = pf.solve_stokes(ind, cfg)
    assert rep.meta["pipeline"] == "cufft-compact"
    ost, ohist, oconv, oit, _ = O.solve_stokes(ind.values, (1.0, 0.0), 1e-6, 1e-6, max_iter=200)
    assert rep.iterations == oit and rep.converged == oconv
    for k in ("u", "u_tilde", "q", "a", "lam"):
        assert rel_l2(getattr(st, k), ost[k]) <= FIELD_TOL, k
    _hist_close(rep.history, ohist)
