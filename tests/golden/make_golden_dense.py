"""Dense-operator golden (reference ``oracle.dense_operators``, src/oracle.py:48-61)
from the LIVE reference, pinning ``oracle/poreflow_oracle.dense_operators``:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_dense.py
"""

import json
import os
import sys
from pathlib import Path

import numpy as np
import scipy

os.environ.setdefault("POREFLOW_BACKEND", "pure")
import poreflow as pf  # noqa: E402  (the reference)
from poreflow.oracle import dense_operators  # noqa: E402

OUT = Path(__file__).resolve().parent

if __name__ == "__main__":
    arrays = {}
    for tag, dims in (("2d", (8, 6)), ("3d", (4, 6, 5))):
        for mode in ("central", "exact"):
            ops = dense_operators(pf.UnitCellGrid(dims), mode)
            arrays[f"{tag}_{mode}_dims"] = np.asarray(dims)
            arrays[f"{tag}_{mode}_grad"] = np.stack(ops.gradient)
            arrays[f"{tag}_{mode}_lap"] = ops.laplacian
    arrays["versions"] = np.asarray(json.dumps({"numpy": np.__version__, "scipy": scipy.__version__,
                                                "python": sys.version.split()[0]}))
    np.savez_compressed(OUT / "dense_ops.npz", **arrays)
    print("wrote dense_ops.npz")
