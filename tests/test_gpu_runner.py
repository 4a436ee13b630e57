"""The run flow on device vs the reference's own ``cli.run`` output
(tests/golden/make_golden_report.py): same report structure and keys, same
iteration counts, tensors and residual rows within round-off, the same output
files with matching contents."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2312_15554_b200 as pf
from paper_2312_15554_b200 import runner

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


def _config(out_dir, sweep=None, fields=("velocity", "concentration", "indicator")):
    return runner.RunConfig(
        geometry=runner.GeometrySpec(kind="disk", radius=0.25, resolution=24),
        stokes=pf.StokesConfig.with_tolerance(1e-6, pressure_gradient=(1.0, 0.5)),
        transport=pf.TransportConfig(pe=10.0, eps=1e-6, composition_gradient=(1.0, 0.0)),
        penalties=pf.PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False),
        output=runner.OutputSpec(out_dir=str(out_dir), fields=tuple(fields), formats=("csv", "vtk")),
        sweep=sweep,
    )


def _compare(ours, gold, path=""):
    if path.endswith("timing") or path.endswith("version"):
        return
    if path.endswith("outputs"):
        assert sorted(Path(f).name for f in ours["files"]) == sorted(Path(f).name for f in gold["files"])
        return
    if isinstance(gold, dict):
        assert set(ours) == set(gold), (path, set(ours) ^ set(gold))
        for k in gold:
            _compare(ours[k], gold[k], f"{path}/{k}")
        return
    if isinstance(gold, list) and any(isinstance(x, (dict, str, list)) for x in gold) and \
            not all(isinstance(x, list) and all(isinstance(y, (int, float)) for y in x) for x in gold):
        assert isinstance(ours, list) and len(ours) == len(gold), path
        for k, (a, b) in enumerate(zip(ours, gold)):
            _compare(a, b, f"{path}[{k}]")
        return
    if isinstance(gold, bool) or isinstance(gold, str) or gold is None:
        assert ours == gold, path
        return
    if isinstance(gold, int):
        assert ours == gold, (path, ours, gold)
        return
    o, g = np.asarray(ours, dtype=float), np.asarray(gold, dtype=float)
    assert o.shape == g.shape, path
    if "/final/" in path:  # residual row of the last iterate: round-off limited
        np.testing.assert_allclose(o, g, rtol=1e-5, atol=0, err_msg=path)
    else:
        scale = float(np.max(np.abs(g))) if g.size else 0.0
        np.testing.assert_allclose(o, g, rtol=1e-9, atol=1e-9 * scale + 1e-15, err_msg=path)


def _rel_close(a, b, tol):
    scale = max(float(np.max(np.abs(b))), 1e-300)
    assert float(np.max(np.abs(a - b))) <= tol * scale


def test_run_matches_reference_report_and_files(tmp_path):
    report, code = runner.run(_config(tmp_path))
    gold_dir = GOLD / "report_disk24"
    gold = json.loads((gold_dir / "report.json").read_text())
    assert code == 0
    ours = json.loads((tmp_path / "report.json").read_text())
    _compare(ours, gold)
    for name in ("flow_history_axis1.csv", "flow_history_axis2.csv", "transport_history_axis1.csv",
                 "transport_history_axis2.csv"):
        a, b = pf.read_history_csv(tmp_path / name), pf.read_history_csv(gold_dir / name)
        assert a.columns == b.columns and a.history.shape == b.history.shape
        for k in range(b.history.shape[1]):
            _rel_close(a.history[:, k], b.history[:, k], 1e-5)
    for name in ("velocity_c0.csv", "velocity_c1.csv", "concentration.csv"):
        a, _ = pf.import_field_csv(tmp_path / name)
        b, _ = pf.import_field_csv(gold_dir / name)
        _rel_close(a, b, 1e-9)
    assert (tmp_path / "indicator.csv").read_text() == (gold_dir / "indicator.csv").read_text()
    va = (tmp_path / "velocity.vtk").read_text().splitlines()
    vb = (gold_dir / "velocity.vtk").read_text().splitlines()
    assert len(va) == len(vb) and [x for x in va if x[:1].isalpha() or x.startswith("#")] == \
        [x for x in vb if x[:1].isalpha() or x.startswith("#")]


@pytest.mark.parametrize("name,sweep", [("report_sweep_b", ("b", (50.0, 200.0))),
                                        ("report_sweep_pe", ("pe", (0.0, 5.0)))])
def test_sweeps_match_reference(tmp_path, name, sweep):
    report, code = runner.run(_config(tmp_path, runner.SweepSpec(*sweep), fields=()))
    gold = json.loads((GOLD / name / "report.json").read_text())
    assert code == 0
    _compare(json.loads((tmp_path / "report.json").read_text()), gold)


def test_run_3d_cell_writes_3d_outputs(tmp_path):
    cfg = runner.RunConfig(
        geometry=runner.GeometrySpec(kind="ball", radius=0.3, resolution=16, dim=3),
        stokes=pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0)),
        transport=pf.TransportConfig(pe=5.0, eps=1e-6, composition_gradient=(1.0, 0.0, 0.0)),
        penalties=pf.PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False),
        output=runner.OutputSpec(out_dir=str(tmp_path), fields=("velocity", "indicator"), formats=("vtk", "npy")))
    report, code = runner.run(cfg)
    assert code == 0
    K = np.asarray(report["effective"]["permeability"])
    assert K.shape == (3, 3) and np.allclose(K, K.T) and np.all(np.diag(K) > 0)
    files = sorted(Path(f).name for f in report["outputs"]["files"])
    assert "velocity.vtk" in files and "velocity.npy" in files and "indicator.npy" in files
    u = np.load(tmp_path / "velocity.npy")
    assert u.shape == (3, 16, 16, 16)
    assert (tmp_path / "velocity.vtk").read_text().splitlines()[4] == "DIMENSIONS 16 16 16"
