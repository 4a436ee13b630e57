"""bench.py's driver contract on CPU: the reference arm (the CPU restatement of
the path, rank 0) prints one JSON line with the required keys; the GPU arm's
keys are checked on the GPU box by the round-end bench itself."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--n", "16", "--steps", "2",
                        "--warmup", "1", "--cpu-budget", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_launcher_fans_out_to_n_ranks():
    """`bench.py --gpus 2` without torchrun starts 2 ranks itself (torch.distributed.run,
    127.0.0.1 rendezvous); the --dry-run probe joins them over gloo on CPU and rank 0
    reports n_gpus = 2 with both ranks present."""
    env = {k: v for k, v in __import__("os").environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run", "--n", "16"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["ranks"] == [0, 1] and d["config"]["cells"] == 2


def test_both_arms_print_the_same_config():
    sys.path.insert(0, str(ROOT))
    import bench

    assert bench.headline_config(256, 1) == bench.headline_config(256, 1)
    src = (ROOT / "bench.py").read_text()
    assert src.count("\"config\": headline_config(") >= 2  # the GPU arm and the reference arm (and the probe)
