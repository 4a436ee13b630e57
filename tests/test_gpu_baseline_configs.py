"""Parity at the BASELINE configurations against the LIVE reference
(tests/golden/make_golden_baseline.py; fields are too large to commit at these
sizes, so the fixtures hold full histories, iteration counts, final penalties,
field norms / maxima and the fields at 4096 fixed voxels).

* cfg 3 — the headline cell: 256^3 random packing (seed 0), reference-default
  ADAPTIVE penalties, eps 1e-5, from zero, truncated by max_iter (40 iterations
  for e1, 8 for e3; residual balancing changes alpha, beta and b inside both
  windows, so the fused pipeline's RSF correction is exercised), on the
  production pipeline the bench times (fused, solid-only storage) and on the
  full-storage fused pipeline.
* cfg 2 — 128^3 sphere array: the stiff converged Stokes solve, then the
  transport solves under that flow at the cfg-2 settings (Pe = 50: the
  reference's own divergence guard trips) and at Pe = 10 (converges).
* cfg 1 — 64^3 sphere array, three load cases with the DEFAULT adaptive
  penalties to convergence, and K.

Bar (north_star): identical iteration counts and flags, fields within 1e-10
relative (sampled voxels against the field's max, norms), final penalties
1e-12, histories by tests/parity_util.py."""

import hashlib
from pathlib import Path

import numpy as np
import pytest

from parity_util import hist_close

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
FIELD_TOL = 1e-10


@pytest.fixture(scope="module")
def pf():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_15554_b200 as pf

    return pf


def load(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def sample_idx(size, k=4096):
    return np.random.default_rng(0).choice(size, size=k, replace=False)  # as make_golden_baseline.py


def check_field(name, x, z, idx):
    ref_s, ref_max, ref_norm = z[f"{name}_sample"], float(z[f"{name}_max"]), float(z[f"{name}_norm"])
    got = np.asarray(x).ravel()[idx]
    err = np.abs(got - ref_s).max() / max(ref_max, 1e-300)
    assert err <= FIELD_TOL, (name, err)
    nrm = float(np.linalg.norm(np.asarray(x)))
    assert abs(nrm - ref_norm) <= FIELD_TOL * max(ref_norm, 1e-300), (name, nrm, ref_norm)


def check_stokes(st, rep, z, n):
    assert rep.iterations == int(z["iterations"])
    assert rep.converged == bool(z["converged"])
    iv, isc = sample_idx(3 * n ** 3), sample_idx(n ** 3)
    for k in ("u", "u_tilde", "a", "lam"):
        check_field(k, getattr(st, k), z, iv)
    check_field("q", st.q, z, isc)
    hist_close(rep.history, z["history"])
    np.testing.assert_allclose(rep.meta["final_penalties"], z["final_penalties"], rtol=1e-12)


@pytest.fixture(scope="module")
def packing256(pf):
    ind = pf.random_packing_geometry(256, seed=0)
    z = load("stokes_packing256_e1_trunc")
    assert hashlib.sha256(np.ascontiguousarray(ind.values).tobytes()).hexdigest() == str(z["ind_sha256"])
    return ind


@pytest.mark.parametrize("compact", [True, False])
@pytest.mark.parametrize("case", ["e1", "e3"])
def test_cfg3_headline_cell_matches_reference(pf, packing256, case, compact):
    z = load(f"stokes_packing256_{case}_trunc")
    cfg = pf.StokesConfig.with_tolerance(float(z["eps"]), pressure_gradient=tuple(float(x) for x in z["g_p"]),
                                         max_iter=int(z["max_iter"]))
    st, rep = pf.solve_stokes_device(packing256, cfg, pf.PenaltyParams(), pipeline="fused", compact=compact)
    assert rep.meta["pipeline"] == ("fused-compact" if compact else "fused")
    # the adaptation must actually have moved the penalties inside the window
    assert np.any(np.asarray(z["final_penalties"]) != 1.0)
    check_stokes(st.to_host(), rep, z, 256)
