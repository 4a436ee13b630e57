"""256^3 truncated solve: fused pipeline vs the cuFFT pipeline (rel-L2 of u, q); a quick parity probe for kernel variants (POREFLOW_B200_LIB)."""
import sys, pathlib; sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
import numpy as np, torch, paper_2312_15554_b200 as pf
ind = pf.random_packing_geometry(256, seed=1)
cfg = pf.StokesConfig.with_tolerance(1e-9, pressure_gradient=(0.3, 1.0, -0.5), max_iter=5)
a, ra = pf.solve_stokes_device(ind, cfg, pipeline="fused")
ua = a.u.cpu().numpy(); qa = a.q.cpu().numpy(); del a; torch.cuda.empty_cache()
b, rb = pf.solve_stokes_device(ind, cfg, pipeline="cufft")
ub = b.u.cpu().numpy(); qb = b.q.cpu().numpy()
print("pipeline", ra.meta["pipeline"], "relL2 u", np.linalg.norm(ua-ub)/np.linalg.norm(ub), "q", np.linalg.norm(qa-qb)/np.linalg.norm(qb))
