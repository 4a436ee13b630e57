"""Host-side logic of the drop-in API (no GPU): config validation, grid and
indicator semantics, symbol tables, the packing generator, backend selection.
Mirrors the reference's own unit tests (tests/test_grid.py, test_stokes.py,
test_transport.py, test_spectral.py) for the pieces that run on the host."""

import numpy as np
from pathlib import Path

import pytest

import paper_2312_15554_b200 as pf
from oracle import poreflow_oracle as O


def test_penalty_and_config_validation():
    with pytest.raises(ValueError):
        pf.PenaltyParams(b=0.0)
    with pytest.raises(ValueError):
        pf.PenaltyParams(growth=(0.9, 1.1, 1.1))
    with pytest.raises(ValueError):
        pf.PenaltyParams(ratio_threshold=(1.0, 10.0, 30.0))
    with pytest.raises(ValueError):
        pf.PenaltyParams(floor=(0.0, 1e-3, 1e-3))
    with pytest.raises(ValueError):
        pf.StokesConfig(nu=0.0)
    with pytest.raises(ValueError):
        pf.StokesConfig(max_iter=0)
    with pytest.raises(ValueError):
        pf.StokesConfig(symbol_mode="upwind")
    for bad in (dict(pe=-1.0), dict(eta=0.0), dict(eta=1.5), dict(a0=0.0), dict(eps=0.0),
                dict(symbol_mode="spectral")):
        with pytest.raises(ValueError):
            pf.TransportConfig(**bad)
    c = pf.StokesConfig.with_tolerance(1e-7)
    assert c.eps_abs == c.eps_rel == 1e-7 and c.symbol_mode == "central"


def test_grid_and_indicator():
    g = pf.UnitCellGrid((8, 16))
    assert g.dim == 2 and g.n_pts == 128 and g.cell_volume == 1.0 / 128
    with pytest.raises(ValueError):
        pf.UnitCellGrid((3, 8))
    with pytest.raises(ValueError):
        pf.IndicatorField(g, np.full((8, 16), 2))
    ind = pf.make_model_geometry(pf.UnitCellGrid((16, 16, 16)), radius=0.25)
    assert np.array_equal(ind.values, O.ball((16, 16, 16), 0.25))
    assert not ind.values.flags.writeable
    assert pf.porosity(ind) == 1.0 - ind.values.mean()
    with pytest.raises(ValueError):
        pf.make_model_geometry(g, radius=0.6)


@pytest.mark.parametrize("mode", ["central", "exact"])
def test_make_symbols_bitwise_equal_to_reference(golden, mode):
    z = golden(f"symbols_{mode}")
    s = pf.make_symbols(pf.UnitCellGrid(tuple(z["dims"])), mode)
    for ax in range(3):
        assert np.array_equal(s.kappa[ax], z[f"k{ax}"])
    assert np.array_equal(s.lap, z["lap"]) and np.array_equal(s.kappa_sq, z["kappa_sq"])


def test_adapt_penalties_branches():
    pen = pf.PenaltyParams()
    P = pf.stokes.ResidualPair
    pairs = (P(100.0, 1, 1.0, 1), P(1.0, 1, 100.0, 1), P(0.0, 1, 0.0, 1))
    out = pf.adapt_penalties(pen, pairs)
    assert out.alpha == pytest.approx(1.1) and out.beta == pytest.approx(1 / 1.1) and out.b == 1.0
    floor = pf.adapt_penalties(pf.PenaltyParams(beta=1e-3), (P(1, 1, 1, 1), P(1.0, 1, 100.0, 1), P(1, 1, 1, 1)))
    assert floor.beta == 1e-3
    grow_inf = pf.adapt_penalties(pen, (P(1.0, 1, 0.0, 1), P(1, 1, 1, 1), P(1, 1, 1, 1)))
    assert grow_inf.alpha == pytest.approx(1.1)


def test_random_packing_generator():
    pk = pf.random_sphere_packing(0)
    assert pk.solid_fraction >= 0.30
    assert pk.radii.min() >= 0.04 and pk.radii.max() <= 0.08
    dv = pk.centers[:, None, :] - pk.centers[None, :, :]
    dv -= np.round(dv)
    d = np.sqrt((dv ** 2).sum(-1))
    rs = pk.radii[:, None] + pk.radii[None, :]
    iu = np.triu_indices(len(pk.radii), 1)
    assert (d[iu] >= rs[iu]).all()  # non-overlapping, minimum image
    ind = pf.rasterize_packing(pk, (32, 32, 32))
    # brute-force minimum-image raster of a few spheres agrees with the boxed one
    grid = ind.grid
    y = grid.meshgrid()
    brute = np.zeros(grid.dims, bool)
    for c, r in zip(pk.centers, pk.radii):
        d2 = 0.0
        for a in range(3):
            dy = y[a] - c[a]
            dy -= np.round(dy)
            d2 = d2 + dy * dy
        brute |= d2 <= r * r
    assert np.array_equal(ind.values.astype(bool), brute)
    assert abs(ind.solid_fraction() - 0.30) < 0.03


def test_backend_selection():
    from paper_2312_15554_b200 import backends

    assert backends.default_backend_name() == "cuda"
    assert backends.kernels_for(3).NAME == "cuda"
    assert backends.HAVE_FUSED is False
    with pytest.raises(ValueError):
        backends.kernels_for(4)


def test_backend_env_rejects_unknown(monkeypatch):
    import importlib

    from paper_2312_15554_b200 import backends

    monkeypatch.setenv("POREFLOW_BACKEND", "upwind")
    with pytest.raises(ValueError):
        importlib.reload(backends)
    monkeypatch.delenv("POREFLOW_BACKEND")
    importlib.reload(backends)


@pytest.mark.parametrize("name", ["pure", "fused", "cuda", "PURE", ""])
def test_backend_env_accepts_reference_names(monkeypatch, name):
    """A process configured for the reference's CPU backends (backends/__init__.py:25-32)
    can import the drop-in: 'pure' / 'fused' select nothing here, the cuda plugin runs."""
    import importlib
    import subprocess
    import sys

    from paper_2312_15554_b200 import backends

    monkeypatch.setenv("POREFLOW_BACKEND", name)
    importlib.reload(backends)
    assert backends.default_backend_name() == "cuda"
    assert backends.kernels_for(3).NAME == "cuda"
    monkeypatch.delenv("POREFLOW_BACKEND")
    importlib.reload(backends)
    # a fresh interpreter importing the whole package with the variable set
    env = dict(__import__("os").environ, POREFLOW_BACKEND=name)
    code = "import paper_2312_15554_b200 as p; assert p.default_backend_name() == 'cuda'"
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=str(Path(__file__).resolve().parents[1]))


def test_packing_slab_rasterization_equals_full_cell():
    """Each slab rank can rasterize only its x-planes (grid.rasterize_packing_slab):
    identical to the corresponding planes of the whole cell, wrap-around included."""
    import numpy as np

    from paper_2312_15554_b200.grid import rasterize_packing, rasterize_packing_slab, random_sphere_packing

    pk = random_sphere_packing(3)
    dims = (32, 28, 24)
    full = rasterize_packing(pk, dims).values
    for lo, hi in [(0, 8), (8, 16), (24, 32), (31, 32)]:
        assert np.array_equal(rasterize_packing_slab(pk, dims, lo, hi), full[lo:hi]), (lo, hi)


def test_pinned_output_policy():
    """device.to_host_many's choice between pinned outputs and the staged ring: the
    first large result is pinned, a later one only when as many pinned result bytes
    have been released (the caller dropped earlier results); small ones always."""
    from paper_2312_15554_b200 import device as D

    saved = dict(D._pin_state)
    try:
        D._pin_state.update(used=False, released=0)
        big = 1 << 30
        assert D._pinned_ok(1 << 20)               # small: always pinned
        assert D._pinned_ok(big)                   # first large result
        assert not D._pinned_ok(big)               # the first still alive: ring
        D._pinned_released(big // 2)
        assert not D._pinned_ok(big)               # not enough released yet
        D._pinned_released(big // 2)
        assert D._pinned_ok(big)                   # the dropped result's blocks are reused
        assert D._pin_state["released"] == 0
    finally:
        D._pin_state.clear()
        D._pin_state.update(saved)
