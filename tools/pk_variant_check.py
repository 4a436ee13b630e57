"""A/B correctness probe for tuning variants: a truncated 256^3 cfg-3 solve (20
iterations, adaptive penalties) with the library POREFLOW_B200_LIB points at;
saves u and the history to OUT.npz, or compares them with REF.npz.

    python tools/pk_variant_check.py OUT.npz [REF.npz]
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2312_15554_b200 as pf

    ind = pf.random_packing_geometry(256, seed=0)
    cfg = pf.StokesConfig.with_tolerance(1e-5, pressure_gradient=(1.0, 0.0, 0.0), max_iter=20)
    st, rep = pf.solve_stokes_device(ind, cfg)
    u = st.u.cpu().numpy()
    np.savez(sys.argv[1], u=u, history=rep.history)
    if len(sys.argv) > 2:
        z = np.load(sys.argv[2])
        du = float(np.linalg.norm(u - z["u"]) / np.linalg.norm(z["u"]))
        dh = float(np.nanmax(np.abs(rep.history - z["history"]) / np.maximum(np.abs(z["history"]), 1e-300)))
        print(f"{sys.argv[1]}: rel|du| {du:.3e} max rel dhist {dh:.3e} {'OK' if du < 1e-12 else 'MISMATCH'}")


if __name__ == "__main__":
    main()
