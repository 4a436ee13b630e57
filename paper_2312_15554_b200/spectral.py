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


# ---------------------------------------------------------------- transforms and
# spectral derivatives (spectral.py:101-143) on the device.  numpy in -> fresh
# numpy out; CUDA tensors in -> CUDA tensors out.  Computed by pf_k_* entry
# points (csrc/pf_ops.cu); there is no host fallback.

def fft(field, grid: UnitCellGrid):
    """Forward transform over the grid axes (leading component axes batched),
    unnormalised, full complex spectrum (spectral.py:101-104)."""
    from . import _devops as D

    host = not D.is_tensor(field)
    dev = D.device_of(field)
    x = D.to_device(np.asarray(field) if host else field, dev)
    return D.out_like(D.fftn_t(x, grid.dim), host)


def ifft(coeffs, grid: UnitCellGrid):
    """Inverse transform with the 1/n factor, truncated to its real part
    (spectral.py:107-115)."""
    from . import _devops as D

    host = not D.is_tensor(coeffs)
    dev = D.device_of(coeffs)
    return D.out_like(D.ifftn_real_t(D.cplx(coeffs, dev), grid.dim), host)


def grad(chi_hat, symbols: SpectralSymbols):
    """Component j = 1j*kappa_j*chi_hat, stacked on a new leading axis (spectral.py:118-124)."""
    from . import _devops as D

    host = not D.is_tensor(chi_hat)
    dev = D.device_of(chi_hat)
    return D.out_like(D.grad_t(D.cplx(chi_hat, dev), D.kappa_tables(symbols, dev), symbols.grid.dim), host)


def div(v_hat, symbols: SpectralSymbols):
    """sum_j 1j*kappa_j*v_hat[j] (spectral.py:127-133)."""
    from . import _devops as D

    host = not D.is_tensor(v_hat)
    dev = D.device_of(v_hat)
    return D.out_like(D.div_t(D.cplx(v_hat, dev), D.kappa_tables(symbols, dev), symbols.grid.dim), host)


def apply_laplacian(chi_hat, symbols: SpectralSymbols):
    """-L(k) * chi_hat (spectral.py:136-138); leading axes of chi_hat are batched."""
    from . import _devops as D

    host = not D.is_tensor(chi_hat)
    dev = D.device_of(chi_hat)
    return D.out_like(D.scale_modes_t(D.real(symbols.lap, dev), D.cplx(chi_hat, dev), -1.0), host)


def gradient_field(field, grid: UnitCellGrid, symbols: SpectralSymbols):
    """Real-space gradient of a real scalar field via the symbol route
    (spectral.py:141-143): ifft(grad(fft(field))), all on the device."""
    from . import _devops as D

    host = not D.is_tensor(field)
    dev = D.device_of(field)
    x = D.real(field, dev)
    g = D.grad_t(D.fftn_t(x, grid.dim), D.kappa_tables(symbols, dev), grid.dim)
    return D.out_like(D.ifftn_real_t(g, grid.dim), host)
