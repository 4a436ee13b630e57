"""Profiling driver: one 256^3 random-packing Stokes cell (bench workload),
W warm-up iterations then K iterations, nothing else — the command that ncu
wraps for the launch list and the per-kernel captures under profiles/.

    python tools/prof_stokes.py [--n 256] [--warmup 3] [--iters 3] [--pipeline auto|fused|cufft]
"""

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--pipeline", default="auto")
    a = ap.parse_args()
    import torch

    import paper_2312_15554_b200 as pf

    dev = torch.device("cuda", 0)
    ind = pf.random_packing_geometry(a.n, seed=0)
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0), max_iter=10**6)
    st = pf.DeviceAdmmState.zeros(ind.grid, dev)
    s = pf.StokesSolver(ind, cfg, pf.PenaltyParams(), st, dev, history_rows=a.warmup + a.iters + 1,
                        pipeline=a.pipeline)
    s.begin()
    s.iterate(a.warmup, poll=False)
    torch.cuda.synchronize()
    s.iterate(a.iters, poll=False)
    torch.cuda.synchronize()
    r = s.end()
    print(f"pipeline={s.pipeline} iterations={r.iterations}")


if __name__ == "__main__":
    main()
