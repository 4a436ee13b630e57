"""How often residual balancing changes b (the RS-fix trigger) in the bench window:
a 256^3 cfg-3 cell, reference-default penalties, iterations 1..K."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2312_15554_b200 as pf  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 320
ind = pf.random_packing_geometry(n, seed=0)
st, rep = pf.solve_stokes_device(ind, pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0), max_iter=K))
h = rep.history
for col, name in ((12, "alpha"), (13, "beta"), (14, "b")):
    ch = np.nonzero(np.diff(h[:, col]) != 0)[0] + 1
    print(f"{name}: {ch.size} changes in {K} iterations; in 10..{K - 10}: {np.sum((ch >= 10) & (ch < K - 10))}; first {ch[:12].tolist()}")
