"""File formats and run-config host logic (no GPU): the writers must reproduce the
reference's own output files byte for byte (fixtures made by the live reference,
tests/golden/make_golden_report.py), and the readers must invert them."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2312_15554_b200 as pf
from paper_2312_15554_b200 import fieldio, runner

G = Path(__file__).parent / "golden" / "report_disk24"


def test_history_csv_matches_reference_bytes(tmp_path):
    for name in ("flow_history_axis1.csv", "transport_history_axis2.csv"):
        rep = pf.read_history_csv(G / name)
        out = pf.write_history_csv(rep, tmp_path / name)
        assert out.read_text() == (G / name).read_text()


def test_field_csv_roundtrip_matches_reference_bytes(tmp_path):
    for name in ("velocity_c0.csv", "velocity_c1.csv", "concentration.csv"):
        data, grid = pf.import_field_csv(G / name)
        assert grid.dims == (24, 24)
    u = np.stack([pf.import_field_csv(G / f"velocity_c{c}.csv")[0] for c in range(2)])
    paths = pf.export_field(u, pf.UnitCellGrid((24, 24)), "csv", tmp_path / "velocity.csv")
    assert [p.name for p in paths] == ["velocity_c0.csv", "velocity_c1.csv"]
    for p in paths:
        assert p.read_text() == (G / p.name).read_text()
    chi, grid = pf.import_field_csv(G / "concentration.csv")
    pf.export_field(chi, grid, "csv", tmp_path / "concentration.csv")
    assert (tmp_path / "concentration.csv").read_text() == (G / "concentration.csv").read_text()


def test_vtk_2d_matches_reference_bytes(tmp_path):
    u = np.stack([pf.import_field_csv(G / f"velocity_c{c}.csv")[0] for c in range(2)])
    pf.export_field(u, pf.UnitCellGrid((24, 24)), "vtk", tmp_path / "velocity.vtk", "velocity")
    assert (tmp_path / "velocity.vtk").read_text() == (G / "velocity.vtk").read_text()
    chi, grid = pf.import_field_csv(G / "concentration.csv")
    pf.export_field(chi, grid, "vtk", tmp_path / "concentration.vtk", "concentration")
    assert (tmp_path / "concentration.vtk").read_text() == (G / "concentration.vtk").read_text()


def test_vtk_3d_layout(tmp_path):
    grid = pf.UnitCellGrid((4, 5, 6))
    f = np.arange(120, dtype=float).reshape(4, 5, 6)
    pf.export_field(f, grid, "vtk", tmp_path / "f.vtk", "f")
    lines = (tmp_path / "f.vtk").read_text().splitlines()
    assert lines[4] == "DIMENSIONS 4 5 6"
    assert lines[7] == "POINT_DATA 120"
    vals = np.array([float(x) for x in lines[10:]])
    # x (first axis) fastest
    assert np.array_equal(vals, np.transpose(f).ravel())


def test_report_json_matches_reference_bytes(tmp_path):
    rep = json.loads((G / "report.json").read_text())
    out = pf.write_report_json(rep, tmp_path / "report.json")
    assert out.read_text() == (G / "report.json").read_text()
    # numpy values encode as the reference's encoder does
    d = {"a": np.arange(3.0), "b": np.float64(0.5), "c": np.int64(2)}
    assert json.loads(pf.write_report_json(d, tmp_path / "x.json").read_text()) == {"a": [0.0, 1.0, 2.0],
                                                                                   "b": 0.5, "c": 2}


def test_indicator_rasters(tmp_path):
    ind = pf.load_indicator_raster(G / "indicator.csv")
    ref = pf.make_model_geometry(pf.UnitCellGrid((24, 24)), radius=0.25)
    assert np.array_equal(ind.values, ref.values)
    assert pf.write_indicator(ind, tmp_path / "indicator.csv").read_text() == (G / "indicator.csv").read_text()
    pgm = pf.write_indicator(ind, tmp_path / "ind.pgm")
    assert np.array_equal(pf.load_indicator_raster(pgm).values, ind.values)
    # 3D: .npy and raw voxel files
    ind3 = pf.make_model_geometry(pf.UnitCellGrid((8, 6, 4)), radius=0.3)
    npy = pf.write_indicator(ind3, tmp_path / "ind3.npy")
    assert np.array_equal(pf.load_indicator_raster(npy).values, ind3.values)
    raw = tmp_path / "ind3.raw"
    (np.asarray(ind3.values, dtype=np.uint8) * 255).tofile(raw)
    back = pf.load_indicator_raw(raw, (8, 6, 4), threshold=128)
    assert back.grid.dims == (8, 6, 4) and np.array_equal(back.values, ind3.values)
    with pytest.raises(ValueError):
        pf.load_indicator_raw(raw, (8, 6, 5))
    with pytest.raises(ValueError):
        pf.write_indicator(ind3, tmp_path / "ind3.csv")
    with pytest.raises(FileNotFoundError):
        pf.load_indicator_raster(tmp_path / "missing.pgm")


def test_run_config_mirrors_reference():
    rep = json.loads((G / "report.json").read_text())
    geo = runner.GeometrySpec(kind="disk", radius=0.25, resolution=24)
    assert geo.describe() == rep["config"]["geometry"]
    assert geo.build().grid.dims == (24, 24)
    cfg = runner.RunConfig(geo, pf.StokesConfig.with_tolerance(1e-6, pressure_gradient=(1.0, 0.5)),
                           pf.TransportConfig(pe=10.0, eps=1e-6, composition_gradient=(1.0, 0.0)),
                           pf.PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False))
    cfgd = json.loads(json.dumps({"stokes": vars(cfg.stokes), "transport": vars(cfg.transport),
                                  "penalties": vars(cfg.penalties)}, cls=fieldio._NumpyEncoder))
    for k in ("stokes", "transport", "penalties"):
        assert cfgd[k] == rep["config"][k]
    with pytest.raises(runner.ConfigError):
        runner.SweepSpec("gamma", (1.0,))
    with pytest.raises(runner.ConfigError):
        runner.GeometrySpec(kind="cube").build()
    assert runner.GeometrySpec(kind="packing", resolution=32, seed=0).build().grid.dims == (32, 32, 32)


def test_packed_indicator_roundtrip(tmp_path):
    """Bit-packed indicator: numpy.packbits order, host values and
    solid fraction equal the byte indicator's, file round trip, validation."""
    import paper_2312_15554_b200 as pf

    for dims in [(13, 7, 5), (16, 16, 16), (9, 11)]:
        rng = np.random.default_rng(sum(dims))
        ind = pf.IndicatorField(pf.UnitCellGrid(dims), (rng.random(dims) < 0.3).astype(np.uint8))
        pk = pf.PackedIndicator.from_indicator(ind)
        assert pk.bits.size == (ind.grid.n_pts + 7) // 8
        assert np.array_equal(pk.values, ind.values) and pk.solid_fraction() == ind.solid_fraction()
        f = pf.save_indicator_bits(pk, tmp_path / "ind.bits")
        back = pf.load_indicator_bits(f, dims)
        assert np.array_equal(back.values, ind.values)
    full = pf.PackedIndicator.from_indicator(pf.IndicatorField(pf.UnitCellGrid((5, 5)), np.ones((5, 5), np.uint8)))
    assert full.all_solid() and full.degenerate
    with pytest.raises(ValueError):
        pf.PackedIndicator(pf.UnitCellGrid((5, 5)), np.zeros(3, np.uint8))  # needs 4 bytes
    with pytest.raises(ValueError):
        pf.PackedIndicator(pf.UnitCellGrid((5, 5)), np.array([0, 0, 0, 0x7F], np.uint8))  # nonzero padding bits
