"""Spectral symbols (setup tables) — mirrors reference ``poreflow.spectral``.

Transform convention (spectral.py:1-21 of the reference): forward unnormalised,
inverse carries 1/n.  The device path never materialises full-grid symbol
arrays: it reads the per-axis tables below (kappa_j and the 1D Laplacian
terms) and forms L = sum_j lap1d_j and kappa_sq = sum_j kappa_j^2 per mode in
the reference's summation order (spectral.py:91-97).  ``make_symbols`` still
returns the full arrays for API compatibility (kernel-plugin callers pass them).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import UnitCellGrid

EXACT = "exact"
CENTRAL = "central"
SYMBOL_MODES = (EXACT, CENTRAL)


def symbol_tables(dims, mode: str):
    """Per-axis (kappa_j, lap1d_j) as spectral.py:78-86 computes them."""
    if mode not in SYMBOL_MODES:
        raise ValueError(f"unknown symbol mode {mode!r}, expected one of {SYMBOL_MODES}")
    out = []
    for n in dims:
        h = 1.0 / n
        k = 2.0 * np.pi * np.fft.fftfreq(n, d=1.0 / n)
        if mode == EXACT:
            kappa, lap1 = k.copy(), k ** 2
        else:
            kappa, lap1 = np.sin(h * k) / h, 4.0 * np.sin(0.5 * h * k) ** 2 / h ** 2
        if n % 2 == 0:
            kappa[n // 2] = 0.0
        out.append((kappa, lap1))
    return out


@dataclass(frozen=True)
class SpectralSymbols:
    """spectral.py:49-69: per-axis kappa, full lap and kappa_sq."""

    grid: UnitCellGrid
    mode: str
    kappa: tuple
    lap: np.ndarray
    kappa_sq: np.ndarray

    def kappa_bc(self, axis: int) -> np.ndarray:
        shape = [1] * self.grid.dim
        shape[axis] = self.grid.dims[axis]
        return self.kappa[axis].reshape(shape)


def make_symbols(grid: UnitCellGrid, mode: str = EXACT) -> SpectralSymbols:
    """spectral.py:72-98 (same default mode, same summation order)."""
    tabs = symbol_tables(grid.dims, mode)
    lap = np.zeros(grid.dims)
    ksq = np.zeros(grid.dims)
    for axis, (kappa, lap1) in enumerate(tabs):
        shape = [1] * grid.dim
        shape[axis] = grid.dims[axis]
        lap += lap1.reshape(shape)
        ksq += kappa.reshape(shape) ** 2
    return SpectralSymbols(grid, mode, tuple(t[0] for t in tabs), lap, ksq)
