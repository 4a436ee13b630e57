"""Fused transport pipeline (pf_fused_transport.cu) against the CPU oracle and
the cuFFT pipeline: identical iteration counts, chi and grad chi within 1e-10
relative L2, divergence guard behaviour, warm start."""

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


@pytest.fixture(scope="module")
def flow64(pf):
    ind = pf.random_packing_geometry(64, seed=4)
    pen = pf.PenaltyParams(alpha=100.0, beta=100.0, b=100.0, adaptive=False)
    st, rep = pf.solve_stokes(ind, pf.StokesConfig.with_tolerance(1e-4, pressure_gradient=(1.0, 0.3, 0.0)), pen)
    return ind, st.u


@pytest.mark.parametrize("pe,a0,g", [(10.0, 0.55, (1.0, 0.0, 0.0)), (50.0, 1.0, (0.0, 1.0, 0.0)),
                                     (0.0, 0.55, (0.3, -0.2, 1.0))])
def test_fused_transport_vs_oracle(pf, flow64, pe, a0, g):
    from oracle import poreflow_oracle as O

    ind, u = flow64
    cfg = pf.TransportConfig(pe=pe, a0=a0, eps=1e-7, composition_gradient=g, max_iter=400)
    st, rep = pf.solve_transport(ind, u, cfg)
    assert rep.meta["pipeline"] == "fused"
    chi, gchi, hist, conv, it, div, b0v = O.solve_transport(ind.values, u, g, pe=pe, a0=a0, eps=1e-7, max_iter=400)
    assert rep.iterations == it and rep.converged == conv and rep.diverged == div
    assert rel_l2(st.chi, chi) <= FIELD_TOL
    assert rel_l2(st.grad_chi, gchi) <= FIELD_TOL
    _hist_close(rep.history, hist)


def test_fused_transport_matches_cufft_pipeline(pf, flow64):
    ind, u = flow64
    cfg = pf.TransportConfig(pe=20.0, eps=1e-8, composition_gradient=(0.0, 0.0, 1.0), max_iter=2000)
    a, ra = pf.solve_transport_device(ind, u, cfg, pipeline="fused")
    b, rb = pf.solve_transport_device(ind, u, cfg, pipeline="cufft")
    assert ra.meta["pipeline"] == "fused" and rb.meta["pipeline"] == "cufft"
    assert ra.converged and rb.converged and ra.iterations == rb.iterations
    assert rel_l2(a.chi.cpu().numpy(), b.chi.cpu().numpy()) <= FIELD_TOL
    assert rel_l2(a.grad_chi.cpu().numpy(), b.grad_chi.cpu().numpy()) <= FIELD_TOL
    _hist_close(ra.history, rb.history)


def test_fused_transport_divergence_guard(pf, flow64):
    from oracle import poreflow_oracle as O

    ind, u = flow64
    cfg = pf.TransportConfig(pe=50.0, a0=0.05, eps=1e-8, composition_gradient=(1.0, 0.0, 0.0), max_iter=500)
    st, rep = pf.solve_transport(ind, u, cfg)
    *_, hist, conv, it, div, _ = O.solve_transport(ind.values, u, (1.0, 0.0, 0.0), pe=50.0, a0=0.05, eps=1e-8,
                                                   max_iter=500)
    assert rep.diverged == div and rep.iterations == it
    _hist_close(rep.history[: min(5, it)], hist[: min(5, it)])


def test_fused_transport_warm_start(pf, flow64):
    from oracle import poreflow_oracle as O

    ind, u = flow64
    rng = np.random.default_rng(2)
    n = 64
    init = pf.TransportState(0.01 * rng.standard_normal((n, n, n)), 0.01 * rng.standard_normal((3, n, n, n)))
    cfg = pf.TransportConfig(pe=5.0, eps=1e-7, composition_gradient=(1.0, 0.0, 0.0), max_iter=12)
    st, rep = pf.solve_transport(ind, u, cfg, init)
    chi, gchi, hist, conv, it, div, _ = O.solve_transport(ind.values, u, (1.0, 0.0, 0.0), pe=5.0, eps=1e-7,
                                                          max_iter=12, init=(init.chi, init.grad_chi))
    assert rep.meta["pipeline"] == "fused" and rep.iterations == it
    assert rel_l2(st.chi, chi) <= FIELD_TOL and rel_l2(st.grad_chi, gchi) <= FIELD_TOL
    _hist_close(rep.history, hist)


@pytest.mark.parametrize("n", [256, 512])
def test_fused_transport_long_matches_cufft_pipeline(pf, n):
    """256^3 (the transport bench size) and 512^3 (long sequences: two 256-point
    blocks + radix-2 stage): truncated solve under a synthetic flow against the
    cuFFT transport pipeline (iterations, chi and grad chi to round-off, history)."""
    import torch

    ind = pf.random_packing_geometry(n, seed=6)
    dev = torch.device("cuda", 0)
    x = torch.arange(n, dtype=torch.float64, device=dev) / n
    u = torch.zeros((3, n, n, n), dtype=torch.float64, device=dev)
    u[0] = 1.0 + 0.2 * torch.sin(2 * np.pi * x)[None, :, None]
    u[1] = 0.1 * torch.cos(2 * np.pi * x)[:, None, None]
    u *= torch.as_tensor(np.asarray(ind.values) == 0, device=dev)
    cfg = pf.TransportConfig(pe=10.0, a0=0.55, eps=1e-12, composition_gradient=(1.0, 0.0, 0.0), max_iter=4)
    a, ra = pf.solve_transport_device(ind, u, cfg, pipeline="fused")
    assert ra.meta["pipeline"] == "fused"
    chi, gchi = a.chi.cpu().numpy(), a.grad_chi.cpu().numpy()
    del a
    torch.cuda.empty_cache()
    b, rb = pf.solve_transport_device(ind, u, cfg, pipeline="cufft")
    assert rb.meta["pipeline"] == "cufft" and ra.iterations == rb.iterations == 4
    assert rel_l2(chi, b.chi.cpu().numpy()) <= FIELD_TOL
    assert rel_l2(gchi, b.grad_chi.cpu().numpy()) <= FIELD_TOL
    _hist_close(ra.history, rb.history)
    del b
    torch.cuda.empty_cache()


def test_fused_transport_256_vs_oracle(pf):
    """The transport bench size on the fused pipeline (256-point whole-row transforms,
    the N = 256 TMA boxes) against the CPU oracle itself, not only the cuFFT pipeline:
    three iterations from zero under a synthetic flow on the seed-6 packing —
    identical iteration count, chi and grad chi within 1e-10 relative L2, history rows."""
    from oracle import poreflow_oracle as O

    n = 256
    ind = pf.random_packing_geometry(n, seed=6)
    x = np.arange(n, dtype=np.float64) / n
    u = np.zeros((3, n, n, n))
    u[0] = 1.0 + 0.2 * np.sin(2 * np.pi * x)[None, :, None]
    u[1] = 0.1 * np.cos(2 * np.pi * x)[:, None, None]
    u *= (np.asarray(ind.values) == 0)
    g = (1.0, 0.0, 0.0)
    cfg = pf.TransportConfig(pe=10.0, a0=0.55, eps=1e-12, composition_gradient=g, max_iter=3)
    st, rep = pf.solve_transport(ind, u, cfg)
    assert rep.meta["pipeline"] == "fused" and rep.iterations == 3
    chi, gchi, hist, conv, it, div, b0v = O.solve_transport(ind.values, u, g, pe=10.0, a0=0.55, eps=1e-12, max_iter=3)
    assert it == 3 and not conv and not div
    assert rel_l2(st.chi, chi) <= FIELD_TOL
    assert rel_l2(st.grad_chi, gchi) <= FIELD_TOL
    np.testing.assert_allclose(rep.meta["b0_vec"], b0v, rtol=1e-12, atol=1e-14)
    _hist_close(rep.history, hist)
