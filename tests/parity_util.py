"""Shared parity checks for the GPU tests (the bar of BASELINE.json's north star)."""

import numpy as np

# Stokes history columns (stokes.py:38-43): residuals at even indices 0..10,
# their tolerances at odd indices 1..11, the penalties alpha, beta, b at 12..14.
STOKES_RESIDUAL_COLS = (0, 2, 4, 6, 8, 10)
STOKES_TOL_COLS = (1, 3, 5, 7, 9, 11)
STOKES_PEN_COLS = (12, 13, 14)


def hist_close(mine, ref, rtol=1e-8, floor=1e-10, tol_rtol=1e-10, pen_rtol=1e-12, kind="stokes"):
    """History rows against a reference history.

    * residual columns: |mine - ref| <= rtol*|ref| + floor*max_rows|ref_col| — every
      entry above ~1e-2 of its column's peak is held to rtol (1e-8); entries far
      below the peak are differences of nearly equal fields (e.g. r_d3 = b|u' - u|
      late in a solve), whose accuracy is bounded by the fields' own round-off, and
      are held to floor x the column's scale instead;
    * tolerance columns (sqrt(n) eps_abs + eps_rel max(...): norms of whole fields,
      well conditioned): tol_rtol;
    * penalty columns (exact products / quotients by the growth factor): pen_rtol.
    For transport histories (r1, r1_tol, r2, r2_tol) pass kind="transport".
    """
    mine, ref = np.asarray(mine), np.asarray(ref)
    assert mine.shape == ref.shape, (mine.shape, ref.shape)
    if kind == "stokes":
        res, tol, pen = STOKES_RESIDUAL_COLS, STOKES_TOL_COLS, STOKES_PEN_COLS
    else:
        res, tol, pen = (0, 2), (1, 3), ()
    scale = np.abs(ref).max(axis=0)
    for cols, rt, fl in ((res, rtol, floor), (tol, tol_rtol, 0.0), (pen, pen_rtol, 0.0)):
        for c in cols:
            bound = rt * np.abs(ref[:, c]) + fl * scale[c] + 1e-300
            err = np.abs(mine[:, c] - ref[:, c])
            bad = np.nonzero(err > bound)[0]
            assert bad.size == 0, (f"history column {c}: row {bad[0]} mine {mine[bad[0], c]!r} "
                                   f"ref {ref[bad[0], c]!r} (|err|/|ref| = {err[bad[0]] / abs(ref[bad[0], c]):.3g})")
