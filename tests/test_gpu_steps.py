"""The reference's step-level API and transform utilities on the device:
``fft``, ``ifft``, ``grad``, ``div``, ``apply_laplacian``, ``gradient_field``
(src/spectral.py:101-143), ``step1_velocity_solve``, ``step2_aux_update``,
``step3_multiplier_update``, ``residuals_and_tolerances`` (src/stokes.py:158-244),
``residual_rhs`` and ``update_concentration`` (src/transport.py:131-177).

The first part ports the reference's own unit tests for these names —
tests/test_spectral.py:15-128, tests/test_stokes.py:37-187 and
tests/test_transport.py:103-166 — with the same inputs, assertions and
tolerances, against the drop-in (dense operators from the CPU oracle's
restatement of src/oracle.py:48-61, pinned in test_oracle_golden.py).  The second
part compares each name with the oracle on seeded 3D inputs.
All calls go through the package API -> C ABI (pf_k_*) -> sm_100a kernels."""

import numpy as np
import pytest

from oracle import poreflow_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_15554_b200 as pf

    return pf


def rel_l2(a, b):
    return float(np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel()) / np.linalg.norm(np.asarray(b).ravel()))


def disk(pf, n, radius=0.25):
    return pf.make_model_geometry(pf.UnitCellGrid((n, n)), radius=radius)


def dense(grid, mode):
    grads, lap = O.dense_operators(grid.dims, mode)
    return grads, lap


# ------------------------------------------------------------ tests/test_spectral.py

def test_constant_field_spectrum_at_zero_only(pf):
    grid = pf.UnitCellGrid((16, 16))
    coeffs = pf.fft(np.full(grid.dims, 3.25), grid)
    assert coeffs[0, 0] == pytest.approx(3.25 * grid.n_pts)
    off = coeffs.copy()
    off[0, 0] = 0.0
    assert np.abs(off).max() < 1e-12 * grid.n_pts


def test_single_harmonic_two_modes(pf):
    grid = pf.UnitCellGrid((16, 16))
    y1, _ = grid.meshgrid()
    mags = np.abs(pf.fft(np.cos(2 * np.pi * y1), grid))
    large = mags > 1e-9 * grid.n_pts
    assert large.sum() == 2
    assert large[1, 0] and large[-1, 0]


def test_round_trip_identity(pf):
    grid = pf.UnitCellGrid((8, 8))
    f = np.random.default_rng(3).standard_normal(grid.dims)
    back = pf.ifft(pf.fft(f, grid), grid)
    assert np.abs(back - f).max() <= 1e-12 * np.abs(f).max()


def test_grad_exact_single_harmonic(pf):
    grid = pf.UnitCellGrid((16, 16))
    y1, _ = grid.meshgrid()
    sym = pf.make_symbols(grid, pf.EXACT)
    g = pf.ifft(pf.grad(pf.fft(np.cos(2 * np.pi * y1), grid), sym), grid)
    assert np.abs(g[0] - (-2 * np.pi * np.sin(2 * np.pi * y1))).max() < 1e-10
    assert np.abs(g[1]).max() < 1e-10


def test_grad_central_amplitude_ratio(pf):
    n, h, k = 16, 1.0 / 16, 2 * np.pi
    ratio = np.sin(h * k) / (h * k)
    assert ratio == pytest.approx(0.9744953584044327, abs=1e-12)
    grid = pf.UnitCellGrid((n, n))
    y1, _ = grid.meshgrid()
    sym = pf.make_symbols(grid, pf.CENTRAL)
    g = pf.ifft(pf.grad(pf.fft(np.cos(k * y1), grid), sym), grid)
    assert np.abs(g[0] - (-k * ratio * np.sin(k * y1))).max() < 1e-10


@pytest.mark.parametrize("mode", ["exact", "central"])
def test_nyquist_derivative_is_exactly_zero(pf, mode):
    grid = pf.UnitCellGrid((16, 16))
    sym = pf.make_symbols(grid, mode)
    nyquist = ((-1.0) ** np.arange(16))[:, None] * np.ones(16)
    g_hat = pf.grad(pf.fft(nyquist, grid), sym)
    assert np.abs(g_hat[0]).max() == 0.0


def test_div_grad_equals_kappa_squared_not_laplacian(pf):
    grid = pf.UnitCellGrid((16, 16))
    sym = pf.make_symbols(grid, pf.CENTRAL)
    f_hat = pf.fft(np.random.default_rng(5).standard_normal(grid.dims), grid)
    composed = pf.div(pf.grad(f_hat, sym), sym)
    direct = -(sym.kappa_bc(0) * (sym.kappa_bc(0) * f_hat))
    direct += -(sym.kappa_bc(1) * (sym.kappa_bc(1) * f_hat))
    assert np.abs(composed - direct).max() == 0.0  # same association: bit-exact
    assert np.abs(sym.kappa_sq - sym.lap).max() > 1.0


def test_div_of_exact_gradient(pf):
    grid = pf.UnitCellGrid((16, 16))
    y1, _ = grid.meshgrid()
    sym = pf.make_symbols(grid, pf.EXACT)
    f = np.cos(2 * np.pi * y1)
    lap_f = pf.ifft(pf.div(pf.grad(pf.fft(f, grid), sym), sym), grid)
    assert np.abs(lap_f - (-(2 * np.pi) ** 2 * f)).max() < 1e-9


def test_div_constant_vector_is_zero(pf):
    grid = pf.UnitCellGrid((16, 16))
    sym = pf.make_symbols(grid, pf.EXACT)
    assert np.abs(pf.div(pf.fft(np.ones((2, *grid.dims)), grid), sym)).max() == 0.0


def test_apply_laplacian_matches_symbol(pf):
    grid = pf.UnitCellGrid((16, 16))
    sym = pf.make_symbols(grid, pf.CENTRAL)
    f_hat = pf.fft(np.random.default_rng(6).standard_normal(grid.dims), grid)
    assert np.abs(pf.apply_laplacian(f_hat, sym) + sym.lap * f_hat).max() == 0.0


@pytest.mark.parametrize("seed,n", [(0, 8), (11, 12), (12345, 16)])
def test_parseval(pf, seed, n):
    grid = pf.UnitCellGrid((n, n))
    f = np.random.default_rng(seed).standard_normal(grid.dims)
    direct = float(np.sum(f ** 2))
    spectral = float(np.sum(np.abs(pf.fft(f, grid)) ** 2)) / grid.n_pts
    assert spectral == pytest.approx(direct, rel=1e-12)


# ------------------------------------------------------------ tests/test_stokes.py

def test_step1_constant_forcing_gives_mean_flow(pf):
    grid = pf.UnitCellGrid((12, 8))
    sym = pf.make_symbols(grid, "central")
    pen = pf.PenaltyParams(alpha=2.0, beta=3.0, b=4.0, adaptive=False)
    cfg = pf.StokesConfig(pressure_gradient=(1.0, 0.0))
    u = pf.step1_velocity_solve(pf.AdmmState.zeros(grid), cfg, pen, sym)
    assert np.abs(u[0] - 0.25).max() < 1e-13
    assert np.abs(u[1]).max() < 1e-13


def test_step1_matches_dense_solve_of_same_system(pf):
    indicator = disk(pf, 8)
    grid = indicator.grid
    cfg = pf.StokesConfig(pressure_gradient=(1.0, 0.0))
    pen = pf.PenaltyParams(alpha=3.0, beta=2.0, b=1.5, adaptive=False)
    sym = pf.make_symbols(grid, cfg.symbol_mode)
    state = pf.AdmmState.zeros(grid)
    u1 = pf.step1_velocity_solve(state, cfg, pen, sym)
    ut1 = pf.step2_aux_update(u1, state, pen, indicator)
    q1, a1, lam1 = pf.step3_multiplier_update(u1, ut1, state, pen, indicator, sym)
    state = pf.AdmmState(u1, ut1, q1, a1, lam1, 1)
    u2 = pf.step1_velocity_solve(state, cfg, pen, sym)

    grads, lap = dense(grid, cfg.symbol_mode)
    n = grid.n_pts
    system = np.zeros((2 * n, 2 * n))
    for c in range(2):
        for m in range(2):
            block = -pen.beta * grads[c] @ grads[m]
            if c == m:
                block = block + cfg.nu * (-lap) + pen.b * np.eye(n)
            system[c * n:(c + 1) * n, m * n:(m + 1) * n] = block
    rhs = np.concatenate([cfg.pressure_gradient[c] - grads[c] @ state.q.ravel() - state.a[c].ravel()
                          + pen.b * state.u_tilde[c].ravel() for c in range(2)])
    u_dense = np.linalg.solve(system, rhs).reshape(2, *grid.dims)
    assert rel_l2(u2, u_dense) < 1e-10


def test_step2_pointwise_cases(pf):
    grid = pf.UnitCellGrid((4, 4))
    indicator = pf.IndicatorField(grid, np.zeros((4, 4), dtype=int))
    pen = pf.PenaltyParams(alpha=1.0, b=1.0, adaptive=False)
    state = pf.AdmmState.zeros(grid)
    u = np.ones((2, 4, 4))
    assert np.allclose(pf.step2_aux_update(u, state, pen, indicator), u)
    solid = pf.IndicatorField(grid, np.ones((4, 4), dtype=int))
    assert np.allclose(pf.step2_aux_update(u, state, pf.PenaltyParams(alpha=3.0, b=1.0), solid), 0.25 * u)
    state.a[0] += 1.0
    state.lam[0] += 3.0
    u2 = np.zeros((2, 4, 4))
    u2[0] = 2.0
    assert np.allclose(pf.step2_aux_update(u2, state, pen, solid), 0.0)


def test_step3_multiplier_updates(pf):
    grid = pf.UnitCellGrid((8, 8))
    sym = pf.make_symbols(grid, "central")
    pen = pf.PenaltyParams(alpha=4.0, beta=2.0, b=2.0, adaptive=False)
    indicator = pf.IndicatorField(grid, np.zeros((8, 8), dtype=int))
    state = pf.AdmmState.zeros(grid)
    u = np.ones((2, 8, 8))
    q, a, lam = pf.step3_multiplier_update(u, u.copy(), state, pen, indicator, sym)
    assert np.abs(q).max() < 1e-14
    assert np.abs(a).max() < 1e-14
    assert np.abs(lam).max() == 0.0
    ut = u.copy()
    ut[0] -= 1.0
    _, a, _ = pf.step3_multiplier_update(u, ut, state, pen, indicator, sym)
    assert np.allclose(a[0], 2.0)
    assert np.allclose(a[1], 0.0)
    solid = pf.IndicatorField(grid, np.ones((8, 8), dtype=int))
    ut = np.zeros((2, 8, 8))
    ut[0] = 0.5
    _, _, lam = pf.step3_multiplier_update(u, ut, state, pen, solid, sym)
    assert np.allclose(lam[0], 2.0)


def test_residuals_zero_state_and_tolerance_floor(pf):
    indicator = disk(pf, 16)
    cfg = pf.StokesConfig(eps_abs=1e-5, eps_rel=1e-5)
    pen = pf.PenaltyParams()
    sym = pf.make_symbols(indicator.grid, cfg.symbol_mode)
    state = pf.AdmmState.zeros(indicator.grid)
    pairs = pf.residuals_and_tolerances(state, state.copy(), pen, cfg, indicator, sym)
    n_vec = state.u.size
    for pair, n in zip(pairs, (n_vec, indicator.grid.n_pts, n_vec)):
        assert pair.primal == 0.0 and pair.dual == 0.0
        assert pair.primal_tol >= np.sqrt(n) * cfg.eps_abs > 0.0
        assert pair.passed


def test_tolerances_reduce_to_absolute_when_eps_rel_zero(pf):
    indicator = disk(pf, 16)
    cfg = pf.StokesConfig(eps_abs=1e-4, eps_rel=0.0)
    pen = pf.PenaltyParams()
    sym = pf.make_symbols(indicator.grid, cfg.symbol_mode)
    rng = np.random.default_rng(9)
    noisy = pf.AdmmState(rng.standard_normal((2, 16, 16)), rng.standard_normal((2, 16, 16)),
                         rng.standard_normal((16, 16)), rng.standard_normal((2, 16, 16)),
                         rng.standard_normal((2, 16, 16)))
    pairs = pf.residuals_and_tolerances(pf.AdmmState.zeros(indicator.grid), noisy, pen, cfg, indicator, sym)
    expect = [np.sqrt(noisy.u.size) * 1e-4, np.sqrt(noisy.q.size) * 1e-4, np.sqrt(noisy.u.size) * 1e-4]
    for pair, tol in zip(pairs, expect):
        assert pair.primal_tol == pytest.approx(tol)
        assert pair.dual_tol == pytest.approx(tol)


# ------------------------------------------------------------ tests/test_transport.py

def pore_only(pf, n):
    grid = pf.UnitCellGrid((n, n))
    return pf.IndicatorField(grid, np.zeros((n, n), dtype=int))


def test_residual_rhs_vanishes_when_medium_matches_comparison(pf):
    indicator = pore_only(pf, 16)
    c = np.array([0.0, 1.0])
    u = np.ones((2, 16, 16)) * c[:, None, None]
    cfg = pf.TransportConfig(pe=3.0, a0=1.0, b0=3.0, composition_gradient=(1.0, 0.0))
    coeffs = pf.build_coefficients(indicator, u, cfg)
    assert np.allclose(coeffs.b0_vec, 3.0 * c)
    sym = pf.make_symbols(indicator.grid, cfg.symbol_mode)
    f_hat = pf.residual_rhs(pf.TransportState.zeros(indicator.grid), coeffs, cfg, sym)
    assert np.abs(f_hat).max() <= 1e-12


def test_residual_rhs_uniform_forcing_is_zero_mode_only(pf):
    indicator = pore_only(pf, 16)
    c = np.array([0.7, 0.3])
    u = np.ones((2, 16, 16)) * c[:, None, None]
    pe = 4.0
    cfg = pf.TransportConfig(pe=pe, a0=1.0, b0=pe * np.linalg.norm(c))
    coeffs = pf.build_coefficients(indicator, u, cfg)
    sym = pf.make_symbols(indicator.grid, cfg.symbol_mode)
    f_hat = pf.residual_rhs(pf.TransportState.zeros(indicator.grid), coeffs, cfg, sym)
    n = indicator.grid.n_pts
    assert f_hat[0, 0] == pytest.approx(n * pe * float(c @ [1.0, 0.0]), rel=1e-12)
    off = f_hat.copy()
    off[0, 0] = 0.0
    assert np.abs(off).max() <= 1e-9 * n


def test_residual_rhs_matches_dense_evaluation(pf):
    rng = np.random.default_rng(21)
    grid = pf.UnitCellGrid((8, 8))
    indicator = pf.IndicatorField(grid, rng.integers(0, 2, size=(8, 8)))
    u = rng.standard_normal((2, 8, 8))
    cfg = pf.TransportConfig(pe=7.0, eta=0.05, a0=0.6, b0=1.0, composition_gradient=(1.0, -0.5))
    sym = pf.make_symbols(grid, cfg.symbol_mode)
    coeffs = pf.build_coefficients(indicator, u, cfg)
    chi = rng.standard_normal((8, 8))
    state = pf.TransportState(chi, pf.gradient_field(chi, grid, sym))
    f_real = pf.ifft(pf.residual_rhs(state, coeffs, cfg, sym), grid)
    grads, _ = dense(grid, cfg.symbol_mode)
    g = np.asarray(cfg.composition_gradient)
    total_grad = [state.grad_chi[c].ravel() + g[c] for c in range(2)]
    expect = coeffs.forcing.ravel().copy()
    for c in range(2):
        expect += grads[c] @ ((coeffs.diffusivity.ravel() - cfg.a0) * total_grad[c])
        expect -= (coeffs.advection[c].ravel() - coeffs.b0_vec[c]) * total_grad[c]
    assert rel_l2(f_real.ravel(), expect) <= 1e-10


def test_update_concentration_poisson_scaling(pf):
    grid = pf.UnitCellGrid((8, 8))
    cfg = pf.TransportConfig(a0=0.7)
    sym = pf.make_symbols(grid, cfg.symbol_mode)
    f_hat = np.zeros(grid.dims, dtype=complex)
    f_hat[2, 1] = 3.0 - 1.0j
    f_hat[-2, -1] = 3.0 + 1.0j
    chi, grad_chi = pf.update_concentration(f_hat, cfg, sym, np.zeros(2))
    chi_hat = pf.fft(chi, grid)
    assert chi_hat[2, 1] == pytest.approx(f_hat[2, 1] / (0.7 * sym.lap[2, 1]), rel=1e-12)
    assert abs(chi_hat[0, 0]) <= 1e-12
    assert np.allclose(grad_chi, pf.gradient_field(chi, grid, sym), atol=1e-13)


def test_update_concentration_zero_rhs(pf):
    grid = pf.UnitCellGrid((8, 8))
    cfg = pf.TransportConfig()
    sym = pf.make_symbols(grid, cfg.symbol_mode)
    chi, grad_chi = pf.update_concentration(np.zeros(grid.dims, dtype=complex), cfg, sym, np.ones(2))
    assert np.abs(chi).max() == 0.0
    assert np.abs(grad_chi).max() == 0.0


def test_update_concentration_solves_uniform_medium_equation(pf):
    grid = pf.UnitCellGrid((8, 8))
    cfg = pf.TransportConfig(a0=0.55)
    b0_vec = np.array([1.0, 0.0])
    sym = pf.make_symbols(grid, cfg.symbol_mode)
    f_hat = np.zeros(grid.dims, dtype=complex)
    f_hat[1, 2] = 2.0 + 0.5j
    f_hat[-1, -2] = 2.0 - 0.5j
    chi, _ = pf.update_concentration(f_hat, cfg, sym, b0_vec)
    grads, lap = dense(grid, cfg.symbol_mode)
    lhs = (-cfg.a0 * lap + b0_vec[0] * grads[0]) @ chi.ravel()
    rhs = pf.ifft(f_hat, grid).ravel()
    assert np.linalg.norm(lhs - rhs) <= 1e-10 * np.linalg.norm(rhs)


# ------------------------------------------------------------ vs the oracle, 3D

@pytest.fixture(scope="module")
def cell3d(pf):
    rng = np.random.default_rng(41)
    dims = (12, 10, 8)
    grid = pf.UnitCellGrid(dims)
    ind = pf.IndicatorField(grid, (rng.random(dims) < 0.3).astype(np.uint8))
    st = pf.AdmmState(*(rng.standard_normal(s) for s in ((3, *dims), (3, *dims), dims, (3, *dims), (3, *dims))))
    return grid, ind, st, rng


@pytest.mark.parametrize("mode", ["central", "exact"])
def test_spectral_utilities_match_oracle_3d(pf, cell3d, mode):
    grid, _, st, rng = cell3d
    sym = pf.make_symbols(grid, mode)
    kap, lap, _ = O.symbols(grid.dims, mode)
    F = pf.fft(st.u, grid)
    ref = O.fftn(st.u, 3)
    assert np.abs(F - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.abs(pf.ifft(ref, grid) - O.ifftn(ref, 3)).max() <= 1e-13 * np.abs(st.u).max()
    Z = rng.standard_normal((3, *grid.dims)) + 1j * rng.standard_normal((3, *grid.dims))
    assert np.array_equal(pf.div(Z, sym), O.spectral_div(Z, kap))  # pointwise: bit-exact
    assert np.array_equal(pf.grad(Z[0], sym), O.spectral_grad(Z[0], kap))
    assert np.array_equal(pf.apply_laplacian(Z, sym), -lap * Z)
    gf = pf.gradient_field(st.q, grid, sym)
    gref = O.ifftn(O.spectral_grad(O.fftn(st.q, 3), kap), 3)
    assert rel_l2(gf, gref) <= 1e-12
    # device tensors in -> device tensors out, same numbers
    import torch

    Fd = pf.fft(torch.from_numpy(st.u).cuda(), grid)
    assert Fd.is_cuda and np.array_equal(Fd.cpu().numpy(), F)


def test_stokes_steps_match_oracle_3d(pf, cell3d):
    grid, ind, st, _ = cell3d
    cfg = pf.StokesConfig(pressure_gradient=(0.3, -1.0, 0.5))
    pen = pf.PenaltyParams(alpha=2.5, beta=1.7, b=3.1, adaptive=False)
    sym = pf.make_symbols(grid, cfg.symbol_mode)
    kap, lap, ksq = O.symbols(grid.dims, cfg.symbol_mode)
    H = ind.as_float()
    u = pf.step1_velocity_solve(st, cfg, pen, sym)
    uh = O.stokes_velocity_update(O.fftn(st.q, 3), O.fftn(st.a, 3), O.fftn(st.u_tilde, 3), kap, lap, ksq,
                                  cfg.nu, pen.beta, pen.b, np.asarray(cfg.pressure_gradient))
    u_ref = O.ifftn(uh, 3)
    assert rel_l2(u, u_ref) <= 1e-12
    ut = pf.step2_aux_update(u_ref, st, pen, ind)
    assert np.array_equal(ut, O.aux_velocity_update(u_ref, st.a, st.lam, H, pen.alpha, pen.b))
    q, a, lam = pf.step3_multiplier_update(u_ref, ut, st, pen, ind, sym)
    a_ref, lam_ref = O.multiplier_update(st.a, st.lam, u_ref, ut, H, pen.alpha, pen.b)
    assert np.array_equal(a, a_ref) and np.array_equal(lam, lam_ref)
    q_ref = st.q - pen.beta * O.ifftn(O.spectral_div(O.fftn(u_ref, 3), kap), 3)
    q_ref -= q_ref.mean()
    assert rel_l2(q, q_ref) <= 1e-12
    assert abs(q.mean()) <= 1e-14 * np.abs(q).max()
    nxt = pf.AdmmState(u_ref, ut, q_ref, a_ref, lam_ref, 1)
    pairs = pf.residuals_and_tolerances(st, nxt, pen, cfg, ind, sym)
    div_p = O.ifftn(O.spectral_div(O.fftn(st.u, 3), kap), 3)
    div_n = O.ifftn(O.spectral_div(O.fftn(u_ref, 3), kap), 3)
    as_dict = lambda x: {k: getattr(x, k) for k in ("u", "u_tilde", "q", "a", "lam")}  # noqa: E731
    ref_pairs = O.stokes_pairs(as_dict(st), as_dict(nxt), div_p, div_n,
                               O.default_penalties(alpha=pen.alpha, beta=pen.beta, b=pen.b),
                               cfg.eps_abs, cfg.eps_rel, H)
    for mine, ref in zip(pairs, ref_pairs):
        got = (mine.primal, mine.primal_tol, mine.dual, mine.dual_tol)
        assert got == pytest.approx(ref, rel=1e-12)


def test_transport_steps_match_oracle_3d(pf, cell3d):
    grid, ind, st, rng = cell3d
    cfg = pf.TransportConfig(pe=6.0, eta=0.05, a0=0.6, b0=1.0, composition_gradient=(0.2, 1.0, -0.4))
    sym = pf.make_symbols(grid, cfg.symbol_mode)
    kap, lap, _ = O.symbols(grid.dims, cfg.symbol_mode)
    coeffs = pf.build_coefficients(ind, st.u, cfg)
    ts = pf.TransportState(st.q, st.a)
    f_hat = pf.residual_rhs(ts, coeffs, cfg, sym)
    w, s = O.transport_polarization(st.a, coeffs.diffusivity, coeffs.advection, coeffs.forcing, cfg.a0,
                                    coeffs.b0_vec, np.asarray(cfg.composition_gradient))
    w_hat, s_hat = O.fftn(w, 3), O.fftn(s, 3)
    f_ref = s_hat
    for c in range(3):
        f_ref = f_ref + 1j * O.axis_table(kap, c, 3) * w_hat[c]
    assert rel_l2(f_hat, f_ref) <= 1e-12
    chi, gch = pf.update_concentration(f_ref, cfg, sym, coeffs.b0_vec)
    ch_ref, gh_ref = O.transport_mode_update(np.zeros((3, *grid.dims), complex), f_ref, kap, lap, cfg.a0,
                                             coeffs.b0_vec)
    assert rel_l2(chi, O.ifftn(ch_ref, 3)) <= 1e-12
    assert rel_l2(gch, O.ifftn(gh_ref, 3)) <= 1e-12
