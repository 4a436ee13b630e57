"""Fused power-of-two pipeline (pf_fused.cu: hand-written axis-split FFTs fused
with the pointwise and spectral steps) against the CPU oracle, the cuFFT
pipeline and the live-reference cfg-1 golden.  Same parity bar: identical
iteration counts, fields within 1e-10 relative L2."""

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
    """Shared bar (tests/parity_util.py): residual columns rtol 1e-8 above the
    round-off floor, tolerance columns 1e-10, penalties 1e-12."""
    from parity_util import hist_close

    hist_close(mine, ref, kind="stokes" if np.shape(ref)[1] == 15 else "transport", **kw)


@pytest.mark.parametrize("compact", [True, False])
@pytest.mark.parametrize("n,iters,geom", [(64, 30, "packing"), (64, 12, "sphere"), (128, 4, "packing")])
def test_fused_truncated_vs_oracle(pf, n, iters, geom, compact):
    from oracle import poreflow_oracle as O

    ind = (pf.random_packing_geometry(n, seed=3) if geom == "packing"
           else pf.make_model_geometry(pf.UnitCellGrid((n, n, n)), radius=0.25))
    g = (0.3, 1.0, -0.5)
    cfg = pf.StokesConfig.with_tolerance(1e-7, pressure_gradient=g, max_iter=iters)
    st, rep = pf.solve_stokes_device(ind, cfg, pipeline="fused", compact=compact)
    assert rep.meta["pipeline"] == ("fused-compact" if compact else "fused")
    ost, ohist, _, oit, ofp = O.solve_stokes(ind.values, g, 1e-7, 1e-7, max_iter=iters)
    assert rep.iterations == oit == iters
    h = st.to_host()
    for k in ("u", "u_tilde", "q", "a", "lam"):
        assert rel_l2(getattr(h, k), ost[k]) <= FIELD_TOL, (k, rel_l2(getattr(h, k), ost[k]))
    _hist_close(rep.history, ohist)
    np.testing.assert_allclose(rep.meta["final_penalties"], ofp, rtol=1e-12)


@pytest.mark.parametrize("compact", [True, False])
def test_fused_128_through_b_changes_vs_oracle(pf, compact):
    """26 iterations of the cfg-3 geometry at 128^3 (seed 0, e1, eps 1e-5, default
    adaptive penalties): residual balancing changes b inside the window (asserted),
    so the RS-fix pass and the axis-1 forward pass's X(u~') correction run — at
    128^3 on the persistent axis-1 kernels (k_m1_pipe)."""
    from oracle import poreflow_oracle as O

    ind = pf.random_packing_geometry(128, seed=0)
    g = (1.0, 0.0, 0.0)
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=g, max_iter=26)
    st, rep = pf.solve_stokes_device(ind, cfg, pipeline="fused", compact=compact)
    assert np.unique(rep.history[:-1, 14]).size > 1
    ost, ohist, _, oit, ofp = O.solve_stokes(ind.values, g, 1e-5, 1e-5, max_iter=26)
    assert rep.iterations == oit == 26
    h = st.to_host()
    for k in ("u", "u_tilde", "q", "a", "lam"):
        assert rel_l2(getattr(h, k), ost[k]) <= FIELD_TOL, (k, rel_l2(getattr(h, k), ost[k]))
    _hist_close(rep.history, ohist)
    np.testing.assert_allclose(rep.meta["final_penalties"], ofp, rtol=1e-12)


def test_fused_matches_cufft_pipeline_full_solve(pf):
    """Converged 64^3 solve (stiff, eps 1e-5): both device pipelines agree."""
    ind = pf.make_model_geometry(pf.UnitCellGrid((64, 64, 64)), radius=0.3)
    pen = pf.PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False)
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(0.0, 0.0, 1.0))
    a, ra = pf.solve_stokes_device(ind, cfg, pen, pipeline="fused")
    b, rb = pf.solve_stokes_device(ind, cfg, pen, pipeline="cufft")
    assert ra.meta["pipeline"] == "fused-compact" and rb.meta["pipeline"] in ("cufft", "cufft-compact")
    assert ra.converged and rb.converged and ra.iterations == rb.iterations
    for k in ("u", "u_tilde", "q", "a", "lam"):
        x, y = getattr(a, k).cpu().numpy(), getattr(b, k).cpu().numpy()
        assert rel_l2(x, y) <= FIELD_TOL, k
    _hist_close(ra.history, rb.history)


def test_fused_warm_start_and_gauge(pf):
    from oracle import poreflow_oracle as O

    n = 64
    ind = pf.random_packing_geometry(n, seed=5)
    rng = np.random.default_rng(1)
    init = pf.AdmmState(*(0.01 * rng.standard_normal(s) for s in [(3, n, n, n), (3, n, n, n), (n, n, n),
                                                                   (3, n, n, n), (3, n, n, n)]))
    g = (1.0, 0.0, 0.0)
    cfg = pf.StokesConfig.with_tolerance(1e-6, pressure_gradient=g, max_iter=10)
    st, rep = pf.solve_stokes(ind, cfg, None, init)
    ost, ohist, _, oit, _ = O.solve_stokes(ind.values, g, 1e-6, 1e-6, max_iter=10,
                                           init=dict(u=init.u, u_tilde=init.u_tilde, q=init.q, a=init.a,
                                                     lam=init.lam))
    assert rep.meta["pipeline"] == "fused" and rep.iterations == oit  # pore a != 0: full storage
    for k in ("u", "u_tilde", "q", "a", "lam"):
        assert rel_l2(getattr(st, k), ost[k]) <= FIELD_TOL, k
    assert abs(st.q.mean()) <= 1e-12 * np.abs(st.q).max()
    _hist_close(rep.history, ohist)


def test_fused_cfg1_sphere64_matches_reference_golden(pf, golden):
    """BASELINE cfg 1 (64^3 sphere array, r = 0.25, stiff, eps 1e-5), 3 load cases:
    iteration counts, history, sampled velocity and the permeability tensor K
    (Stokes symbols) against the live reference."""
    import os

    path = os.path.join(os.path.dirname(__file__), "golden", "stokes_sphere64_cfg1.npz")
    if not os.path.exists(path):
        pytest.skip("cfg-1 golden not generated")
    z = golden("stokes_sphere64_cfg1")
    n = int(z["dims"][0])
    solid = np.unpackbits(z["solid_packed"])[: n ** 3].reshape(n, n, n)
    ind = pf.IndicatorField(pf.UnitCellGrid((n, n, n)), solid)
    pen = pf.PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False)
    us = []
    for ax in range(3):
        g = [0.0] * 3
        g[ax] = 1.0
        st, rep = pf.solve_stokes(ind, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=tuple(g)), pen)
        assert rep.meta["pipeline"] == "fused-compact"
        assert rep.iterations == int(z["iterations"][ax])
        ref_h = z["history"][ax][: rep.iterations]
        _hist_close(rep.history, ref_h)
        us_s = st.u.ravel()[z["sample"]]
        assert np.abs(us_s - z["u_sample"][ax]).max() <= 1e-10 * z["u_max"][ax]
        assert abs(np.linalg.norm(st.u) - z["u_norm"][ax]) <= 1e-10 * z["u_norm"][ax]
        us.append(st.u)
    K = pf.permeability(us, ind, pf.make_symbols(ind.grid, "central"))
    assert np.abs(K - z["K"]).max() <= 1e-9 * np.abs(z["K"]).max()


def test_fused_pipelines_bitwise_deterministic(pf):
    """Race detector (compute-sanitizer is closed on this pool): the hand-written
    kernels use warp-synchronous shared-memory FFTs, TMA/LDGSTS staging and
    fixed-order reductions, so repeated solves must agree to the last bit
    (the reference's own determinism contract, tests/test_backends.py:92-98)."""
    ind = pf.random_packing_geometry(64, seed=11)
    cfg = pf.StokesConfig.with_tolerance(1e-6, pressure_gradient=(0.2, 1.0, 0.0), max_iter=25)
    a, ra = pf.solve_stokes_device(ind, cfg, pipeline="fused")
    b, rb = pf.solve_stokes_device(ind, cfg, pipeline="fused")
    assert ra.meta["pipeline"] == "fused-compact"
    assert np.array_equal(ra.history, rb.history)
    for k in ("u", "u_tilde", "q", "a", "lam"):
        assert bool((getattr(a, k) == getattr(b, k)).all()), k
    tc = pf.TransportConfig(pe=10.0, eps=1e-9, composition_gradient=(0.0, 1.0, 0.0), max_iter=15)
    x, rx = pf.solve_transport_device(ind, a.u, tc, pipeline="fused")
    y, ry = pf.solve_transport_device(ind, a.u, tc, pipeline="fused")
    assert np.array_equal(rx.history, ry.history)
    assert bool((x.chi == y.chi).all()) and bool((x.grad_chi == y.grad_chi).all())


def test_fused_exact_symbols_vs_oracle(pf):
    from oracle import poreflow_oracle as O

    ind = pf.make_model_geometry(pf.UnitCellGrid((64, 64, 64)), radius=0.3)
    cfg = pf.StokesConfig.with_tolerance(1e-7, pressure_gradient=(0.0, 0.0, 1.0), max_iter=10, symbol_mode="exact")
    st, rep = pf.solve_stokes(ind, cfg)
    assert rep.meta["pipeline"] == "fused-compact"
    ost, ohist, _, oit, _ = O.solve_stokes(ind.values, (0.0, 0.0, 1.0), 1e-7, 1e-7, max_iter=10, mode="exact")
    for k in ("u", "u_tilde", "q", "a", "lam"):
        assert rel_l2(getattr(st, k), ost[k]) <= FIELD_TOL, k
    _hist_close(rep.history, ohist)


def test_compact_warm_start_continues_exactly(pf):
    """A state produced by the compact path (pore a == 0 exactly) warm-starts the
    compact path again; the two halves equal one uninterrupted run."""
    ind = pf.random_packing_geometry(64, seed=12)
    g = (1.0, 0.0, 0.5)
    full, rf = pf.solve_stokes_device(ind, pf.StokesConfig.with_tolerance(1e-7, pressure_gradient=g, max_iter=20))
    half, rh = pf.solve_stokes_device(ind, pf.StokesConfig.with_tolerance(1e-7, pressure_gradient=g, max_iter=10))
    assert float(half.a[:, torch_pore(ind, half.a)].abs().max()) == 0.0
    rest, rr = pf.solve_stokes_device(ind, pf.StokesConfig.with_tolerance(1e-7, pressure_gradient=g, max_iter=10),
                                      pf.PenaltyParams(*rh.meta["final_penalties"]), init=half)
    assert rr.meta["pipeline"] == "fused-compact"
    for k in ("u", "u_tilde", "a", "lam"):
        assert rel_l2(getattr(rest, k).cpu().numpy(), getattr(full, k).cpu().numpy()) <= 1e-12, k


def torch_pore(ind, like):
    import torch

    return torch.from_numpy(ind.values == 0).to(like.device)


@pytest.mark.parametrize("compact", [True, False])
def test_fused_long_sequences_512_match_cufft_pipeline(pf, compact):
    """N = 512: every axis transform is two 256-point block transforms plus a
    radix-2 stage (pf_fft.cuh radix_stage / fft_units).  A truncated adaptive
    solve on the fused pipeline agrees with the cuFFT pipeline (iterations,
    fields to round-off, history)."""
    import torch

    ind = pf.random_packing_geometry(512, seed=2)
    cfg = pf.StokesConfig.with_tolerance(1e-9, pressure_gradient=(0.3, 1.0, -0.5), max_iter=4)
    a, ra = pf.solve_stokes_device(ind, cfg, pipeline="fused", compact=compact)
    assert ra.meta["pipeline"] == ("fused-compact" if compact else "fused")
    ah = {k: getattr(a, k).cpu().numpy() for k in ("u", "u_tilde", "q", "a", "lam")}
    del a
    torch.cuda.empty_cache()
    b, rb = pf.solve_stokes_device(ind, cfg, pipeline="cufft")
    assert rb.meta["pipeline"] in ("cufft", "cufft-compact") and ra.iterations == rb.iterations == 4
    for k in ("u", "u_tilde", "q", "a", "lam"):
        assert rel_l2(ah[k], getattr(b, k).cpu().numpy()) <= FIELD_TOL, k
    _hist_close(ra.history, rb.history)
    del b
    torch.cuda.empty_cache()


def test_fused_256_headline_cell_matches_cufft_pipeline(pf):
    """The bench's own size (256^3 random packing, compact storage, whole-warp RS
    transforms, TMA pencils): a truncated adaptive solve equals the cuFFT
    pipeline's to round-off."""
    import torch

    ind = pf.random_packing_geometry(256, seed=1)
    cfg = pf.StokesConfig.with_tolerance(1e-9, pressure_gradient=(0.3, 1.0, -0.5), max_iter=5)
    a, ra = pf.solve_stokes_device(ind, cfg, pipeline="fused")
    assert ra.meta["pipeline"] == "fused-compact"
    ah = {k: getattr(a, k).cpu().numpy() for k in ("u", "u_tilde", "q", "a", "lam")}
    del a
    torch.cuda.empty_cache()
    b, rb = pf.solve_stokes_device(ind, cfg, pipeline="cufft")
    assert ra.iterations == rb.iterations == 5
    for k in ("u", "u_tilde", "q", "a", "lam"):
        assert rel_l2(ah[k], getattr(b, k).cpu().numpy()) <= FIELD_TOL, k
    _hist_close(ra.history, rb.history)
    del b
    torch.cuda.empty_cache()
