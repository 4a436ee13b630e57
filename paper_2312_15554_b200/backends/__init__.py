"""Kernel plugin selection — mirrors reference ``poreflow.backends``
(pkg/src/poreflow/backends/__init__.py:17-54).

The reference ships ``pure`` (numpy, any d) and ``fused`` (Cython, 2D).  This
package ships exactly one implementation, ``cuda`` (sm_100a, any d <= 3), and
no fallback: ``POREFLOW_BACKEND`` may be empty, ``cuda``, or one of the
reference's names (``pure``, ``fused``), which select nothing here; anything
else is a ValueError, and a missing native library raises ImportError at first use.
"""

from __future__ import annotations

import os

from . import cuda

# The reference accepts "", "pure" and "fused" (backends/__init__.py:25-32).  A process
# configured for the reference's CPU backends must still be able to import this
# package, so those names are accepted and simply do not select anything here:
# every grid runs on the ``cuda`` plugin.  Unknown names raise, as in the reference.
_KNOWN = ("", "cuda", "pure", "fused")
_requested = os.environ.get("POREFLOW_BACKEND", "").strip().lower()
if _requested not in _KNOWN:
    raise ValueError(f"POREFLOW_BACKEND must be one of 'cuda', 'pure', 'fused' or empty, got {_requested!r}")

HAVE_FUSED = False  # the reference's 2D Cython extension has no counterpart here
HAVE_CUDA = True


def default_backend_name() -> str:
    return "cuda"


def kernels_for(dim: int):
    """Kernel module for a grid of the given dimension (1 <= dim <= 3)."""
    if not 1 <= dim <= 3:
        raise ValueError(f"cuda kernels support 1 <= dim <= 3, got {dim}")
    return cuda


def num_threads() -> int:
    """Kept for signature compatibility (backends/__init__.py:50-54); unused on device."""
    cap = os.environ.get("POREFLOW_THREADS", "").strip()
    if cap:
        return max(1, int(cap))
    return max(1, os.cpu_count() or 1)
