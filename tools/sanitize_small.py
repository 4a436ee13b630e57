"""Small fused Stokes + transport solves and the cuFFT / slab pipelines on 64^3 and
odd grids — the workload compute-sanitizer runs (memcheck / racecheck)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2312_15554_b200 as pf  # noqa: E402
from paper_2312_15554_b200.slab import solve_stokes_slab  # noqa: E402

ind = pf.random_packing_geometry(64, seed=1)
cfg = pf.StokesConfig.with_tolerance(1e-6, pressure_gradient=(1.0, 0.0, 0.0), max_iter=3)
st, rep = pf.solve_stokes_device(ind, cfg, pipeline="fused")
st2, rep2 = pf.solve_stokes_device(ind, cfg, pipeline="cufft")
ts, trep = pf.solve_transport_device(ind, st.u, pf.TransportConfig(pe=5.0, composition_gradient=(1.0, 0, 0),
                                                                   max_iter=3), pipeline="fused")
odd = pf.IndicatorField(pf.UnitCellGrid((10, 12, 9)), (np.random.default_rng(0).random((10, 12, 9)) < 0.2))
st3, rep3 = pf.solve_stokes(odd, pf.StokesConfig.with_tolerance(1e-6, pressure_gradient=(1.0, 0, 0), max_iter=3))
sl, srep = solve_stokes_slab(odd.values, odd.grid.dims, pf.StokesConfig.with_tolerance(1e-6, pressure_gradient=(1.0, 0, 0), max_iter=3))
K = pf.permeability([st.u, st.u, st.u], ind, "central")
torch.cuda.synchronize()
print("ok", rep.iterations, rep2.iterations, trep.iterations, rep3.iterations, srep.iterations)
