"""Profiling driver: the bench transport workload (n^3 sphere array, r = 0.25,
Pe = 10) -- a short Stokes solve for the flow, then W warm-up and K transport
iterations, nothing else; the command ncu wraps for the transport captures.

    python tools/prof_transport.py [--n 256] [--warmup 3] [--iters 3]
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
    a = ap.parse_args()
    import torch

    import paper_2312_15554_b200 as pf

    dev = torch.device("cuda", 0)
    n = a.n
    ind = pf.make_model_geometry(pf.UnitCellGrid((n, n, n)), radius=0.25)
    pen = pf.PenaltyParams(alpha=100.0, beta=100.0, b=100.0, adaptive=False)
    st, _ = pf.solve_stokes_device(ind, pf.StokesConfig.with_tolerance(1e-4, pressure_gradient=(1.0, 0.0, 0.0),
                                                                       max_iter=20), pen)
    cfg = pf.TransportConfig(pe=10.0, a0=0.55, eps=1e-12, composition_gradient=(1.0, 0.0, 0.0), max_iter=10**6)
    z = lambda *s: torch.zeros(s, dtype=torch.float64, device=dev)  # noqa: E731
    state = pf.DeviceTransportState(z(n, n, n), z(3, n, n, n))
    s = pf.TransportSolver(ind, st.u, cfg, state, dev, history_rows=a.warmup + a.iters + 4)
    s.begin()
    s.iterate(a.warmup, poll=False)
    torch.cuda.synchronize()
    s.iterate(a.iters, poll=False)
    torch.cuda.synchronize()
    r = s.end()
    print(f"pipeline={s.pipeline} iterations={r.iterations}")


if __name__ == "__main__":
    main()
