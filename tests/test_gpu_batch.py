"""Concurrent independent solves on one GPU (batch.py) return bit-for-bit the
sequential results: each solve keeps its own plan, stream, kernels and
reduction order; only the host's issue order changes."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_15554_b200 as pf

    return pf


def _unit(d, ax):
    g = [0.0] * d
    g[ax] = 1.0
    return tuple(g)


@pytest.mark.parametrize("dims,adaptive", [((64, 64, 64), True), ((64, 64, 64), False), ((20, 18, 16), True),
                                           ((32, 24), True)])
def test_stokes_batch_bitwise_equals_sequential(pf, dims, adaptive):
    from paper_2312_15554_b200.batch import solve_stokes_many_device

    d = len(dims)
    ind = pf.make_model_geometry(pf.UnitCellGrid(dims), radius=0.3)
    pen = pf.PenaltyParams() if adaptive else pf.PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False)
    cfgs = [pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=_unit(d, ax), max_iter=300) for ax in range(d)]
    seq = [pf.solve_stokes_device(ind, c, pen) for c in cfgs]
    bat = solve_stokes_many_device([ind] * d, cfgs, pen)
    for (s1, r1), (s2, r2) in zip(seq, bat):
        assert r1.iterations == r2.iterations and r1.converged == r2.converged
        assert np.array_equal(r1.history, r2.history)
        for k in ("u", "u_tilde", "q", "a", "lam"):
            assert bool((getattr(s1, k) == getattr(s2, k)).all()), k


def test_stokes_batch_mixed_cells_and_all_solid(pf):
    from paper_2312_15554_b200.batch import solve_stokes_many_device

    g = pf.UnitCellGrid((64, 64, 64))
    inds = [pf.random_packing_geometry(64, seed=s) for s in range(3)]
    inds.append(pf.IndicatorField(g, np.ones(g.dims, dtype=np.uint8)))
    cfg = pf.StokesConfig.with_tolerance(1e-4, pressure_gradient=(1.0, 0.0, 0.0), max_iter=500)
    bat = solve_stokes_many_device(inds, [cfg] * 4)
    for ind, (st, rep) in zip(inds[:3], bat[:3]):
        s1, r1 = pf.solve_stokes_device(ind, cfg)
        assert r1.iterations == rep.iterations
        assert bool((s1.u == st.u).all())
    fast = pf.solve_stokes_device(inds[3], cfg)[1]  # the reference's all-solid fast path
    assert bat[3][1].converged and bat[3][1].iterations == fast.iterations
    assert np.array_equal(bat[3][1].history, fast.history) and float(bat[3][0].u.abs().max()) == 0.0


@pytest.mark.parametrize("dims", [(64, 64, 64), (20, 18, 16)])
def test_transport_batch_bitwise_equals_sequential(pf, dims):
    from paper_2312_15554_b200.batch import solve_transport_many_device

    d = len(dims)
    ind = pf.make_model_geometry(pf.UnitCellGrid(dims), radius=0.3)
    st, _ = pf.solve_stokes_device(ind, pf.StokesConfig.with_tolerance(1e-4, pressure_gradient=_unit(d, 0)),
                                   pf.PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False))
    cfgs = [pf.TransportConfig(pe=10.0, eps=1e-6, composition_gradient=_unit(d, ax)) for ax in range(d)]
    seq = [pf.solve_transport_device(ind, st.u, c) for c in cfgs]
    bat = solve_transport_many_device([ind] * d, [st.u] * d, cfgs)
    for (s1, r1), (s2, r2) in zip(seq, bat):
        assert r1.iterations == r2.iterations and r1.converged == r2.converged
        assert np.array_equal(r1.history, r2.history)
        assert bool((s1.chi == s2.chi).all()) and bool((s1.grad_chi == s2.grad_chi).all())


def test_solver_instances_on_host_threads(pf):
    """The reference's concurrency contract (tests/test_backends.py:131-149):
    independent solves issued from several host threads at once (each thread
    its own plans and current stream) equal the same solves run one by one."""
    import threading

    import torch

    cells = [pf.random_packing_geometry(48, seed=s) for s in range(3)]
    cfg = pf.StokesConfig.with_tolerance(1e-6, pressure_gradient=(1.0, 0.0, 0.0), max_iter=80)
    tcfg = pf.TransportConfig(pe=5.0, eps=1e-8, composition_gradient=(0.0, 1.0, 0.0), max_iter=40)
    seq = []
    for ind in cells:
        st, rep = pf.solve_stokes(ind, cfg)
        ts, trep = pf.solve_transport(ind, st.u, tcfg)
        seq.append((st.u, rep.iterations, ts.chi, trep.iterations))
    out, errs = [None] * len(cells), []

    def work(k):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                st, rep = pf.solve_stokes(cells[k], cfg)
                ts, trep = pf.solve_transport(cells[k], st.u, tcfg)
            out[k] = (st.u, rep.iterations, ts.chi, trep.iterations)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(cells))]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    for a, b in zip(seq, out):
        assert a[1] == b[1] and a[3] == b[3]
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2])


@pytest.mark.parametrize("n", [64, 128])
def test_stokes_batch_different_cells_through_b_changes(pf, n):
    """Several packings (different solid staging capacities per plan) solved
    concurrently through residual-balancing changes of b: every cell's RS-fix launch
    must fit the per-function shared-memory limit whichever plan set it last (the
    cfg-4 ensemble bench hit a launch failure before the limit was set to the worst
    case), and each result equals its own sequential solve bit for bit."""
    from paper_2312_15554_b200.batch import solve_stokes_many_device

    inds = [pf.random_packing_geometry(n, seed=s) for s in (0, 5, 9, 17)]
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0), max_iter=26)
    bat = solve_stokes_many_device(inds, [cfg] * len(inds))
    changed = 0
    for ind, (st, rep) in zip(inds, bat):
        s1, r1 = pf.solve_stokes_device(ind, cfg)
        assert r1.iterations == rep.iterations == 26
        assert np.array_equal(r1.history, rep.history)
        assert bool((s1.u == st.u).all())
        changed += int(np.unique(rep.history[:-1, 14]).size > 1)
    assert changed >= 1
