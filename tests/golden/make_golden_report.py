"""Report / file-format goldens from the LIVE reference's run flow
(pkg/src/poreflow/cli.py:282-414, fieldio.py): a 2D disk cell run end to end with
every output (report.json, history CSVs, velocity / concentration / indicator
fields as CSV and VTK), a stiff-penalty sweep and a transport-parameter sweep.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_report.py
"""

import os
import shutil
import sys
from pathlib import Path

os.environ.setdefault("POREFLOW_BACKEND", "pure")
from poreflow import cli  # noqa: E402  (the reference)
from poreflow.stokes import PenaltyParams, StokesConfig  # noqa: E402
from poreflow.transport import TransportConfig  # noqa: E402

OUT = Path(__file__).resolve().parent


def config(out_dir, sweep=None, fields=("velocity", "concentration", "indicator")):
    return cli.RunConfig(
        geometry=cli.GeometrySpec(kind="disk", radius=0.25, resolution=24),
        stokes=StokesConfig.with_tolerance(1e-6, pressure_gradient=(1.0, 0.5)),
        transport=TransportConfig(pe=10.0, eps=1e-6, composition_gradient=(1.0, 0.0)),
        penalties=PenaltyParams(alpha=1000.0, beta=1000.0, b=1000.0, adaptive=False),  # tests/helpers.py:32-35
        output=cli.OutputSpec(out_dir=str(out_dir), fields=tuple(fields), formats=("csv", "vtk"), histories=True),
        sweep=sweep,
    )


def main():
    runs = {
        "report_disk24": config(OUT / "report_disk24"),
        "report_sweep_b": config(OUT / "report_sweep_b", cli.SweepSpec("b", (50.0, 200.0)), fields=()),
        "report_sweep_pe": config(OUT / "report_sweep_pe", cli.SweepSpec("pe", (0.0, 5.0)), fields=()),
    }
    for name, cfg in runs.items():
        d = OUT / name
        if d.exists():
            shutil.rmtree(d)
        report, code = cli.run(cfg)
        print(name, "exit", code, sorted(report))
    return 0


if __name__ == "__main__":
    sys.exit(main())
