import time, numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2312_15554_b200 as pf
n=256
ind0 = pf.random_packing_geometry(n, seed=0)
vals = np.array(ind0.values)
cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0,0,0), max_iter=300)
pf.solve_stokes(pf.IndicatorField(pf.UnitCellGrid((n,n,n)), vals), pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0,0,0), max_iter=5))
torch.cuda.synchronize()
t0=time.perf_counter(); ind = pf.IndicatorField(pf.UnitCellGrid((n,n,n)), vals); t1=time.perf_counter()
st, rep = pf.solve_stokes_device(ind, cfg); torch.cuda.synchronize(); t2=time.perf_counter()
h = st.to_host(); t3=time.perf_counter()
print(f"indicator {t1-t0:.3f}s  device solve {t2-t1:.3f}s  to_host {t3-t2:.3f}s")
x = st.u
for k in range(2):
    t=time.perf_counter(); p = torch.empty(x.shape, dtype=x.dtype, pin_memory=True); t_alloc=time.perf_counter()-t
    t=time.perf_counter(); p.copy_(x, non_blocking=True); torch.cuda.synchronize(); t_cp=time.perf_counter()-t
    print(f"pinned alloc {t_alloc:.3f}s copy {t_cp:.3f}s ({x.numel()*8/t_cp/1e9:.1f} GB/s)")
t=time.perf_counter(); y=x.cpu(); print(f"pageable .cpu() {time.perf_counter()-t:.3f}s")
