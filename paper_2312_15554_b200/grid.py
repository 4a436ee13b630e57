"""Periodic unit-cell grids, the solid indicator and synthetic microstructures.

Mirrors reference ``poreflow.grid`` (pkg/src/poreflow/grid.py:25-131): a
structured periodic grid over the unit cube sampled at cell centres
``y_j = (i + 1/2)/N_j``; the indicator is 1 on solid, 0 on pore and is
immutable.  Adds the 3D random polydisperse sphere packing that BASELINE
configs 3-5 name, which the reference does not ship.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MIN_CELLS_PER_AXIS = 4  # grid.py:22


@dataclass(frozen=True)
class UnitCellGrid:
    """grid.py:25-71."""

    dims: tuple[int, ...]

    def __post_init__(self):
        dims = tuple(int(n) for n in np.atleast_1d(np.asarray(self.dims, dtype=int)))
        object.__setattr__(self, "dims", dims)
        if not dims:
            raise ValueError("grid needs at least one axis")
        if any(n < MIN_CELLS_PER_AXIS for n in dims):
            raise ValueError(f"need at least {MIN_CELLS_PER_AXIS} cells per axis, got {dims}")

    @property
    def dim(self) -> int:
        return len(self.dims)

    @property
    def spacing(self) -> tuple[float, ...]:
        return tuple(1.0 / n for n in self.dims)

    @property
    def n_pts(self) -> int:
        return int(np.prod(self.dims))

    @property
    def cell_volume(self) -> float:
        return float(np.prod(self.spacing))

    def axis_centers(self, axis: int) -> np.ndarray:
        n = self.dims[axis]
        return (np.arange(n) + 0.5) / n

    def meshgrid(self) -> tuple[np.ndarray, ...]:
        return tuple(np.meshgrid(*(self.axis_centers(a) for a in range(self.dim)), indexing="ij"))

    def zeros_scalar(self) -> np.ndarray:
        return np.zeros(self.dims)

    def zeros_vector(self) -> np.ndarray:
        return np.zeros((self.dim, *self.dims))


@dataclass(frozen=True)
class IndicatorField:
    """Solid indicator, uint8 0/1, read-only.  grid.py:74-105."""

    grid: UnitCellGrid
    values: np.ndarray
    _device_cache: dict = field(default_factory=dict, init=False, repr=False, compare=False)

    def __post_init__(self):
        values = np.asarray(self.values)
        if values.shape != self.grid.dims:
            raise ValueError(f"indicator shape {values.shape} does not match grid {self.grid.dims}")
        if values.dtype == np.bool_ or values.size == 0:
            ok = True
        elif np.issubdtype(values.dtype, np.unsignedinteger):
            ok = int(values.max()) <= 1  # one pass instead of two comparison temporaries
        elif np.issubdtype(values.dtype, np.integer):
            ok = int(values.min()) >= 0 and int(values.max()) <= 1
        else:
            ok = bool(((values == 0) | (values == 1)).all())
        if not ok:
            raise ValueError("indicator values must be exactly 0 or 1")
        values = values.astype(np.uint8)
        values.setflags(write=False)
        object.__setattr__(self, "values", values)

    def solid_fraction(self) -> float:
        return float(self.values.mean())

    @property
    def degenerate(self) -> bool:
        frac = self.solid_fraction()
        return frac == 0.0 or frac == 1.0

    def as_float(self) -> np.ndarray:
        return self.values.astype(np.float64)


class PackedIndicator:
    """Bit-packed solid indicator: 1 bit per voxel in numpy.packbits
    order (the first voxel, C order, in the most significant bit of byte 0).
    Accepted wherever an ``IndicatorField`` is: the device solvers copy the
    ceil(n / 8) bytes to the GPU and unpack them there (``pf_unpack_bits``);
    ``values`` unpacks on the host only for host consumers (cached)."""

    def __init__(self, grid: UnitCellGrid, bits):
        bits = np.ascontiguousarray(np.asarray(bits, dtype=np.uint8).ravel())
        n = grid.n_pts
        if bits.size != (n + 7) // 8:
            raise ValueError(f"packed indicator needs {(n + 7) // 8} bytes for grid {grid.dims}, got {bits.size}")
        if n % 8 and int(bits[-1]) & ((1 << (8 - n % 8)) - 1):
            raise ValueError("padding bits of the last byte must be zero")
        bits.setflags(write=False)
        self.grid, self.bits = grid, bits
        self._values = None
        self._device_cache: dict = {}

    @classmethod
    def from_indicator(cls, indicator: IndicatorField) -> "PackedIndicator":
        return cls(indicator.grid, np.packbits(np.asarray(indicator.values, dtype=np.uint8).ravel()))

    @property
    def values(self) -> np.ndarray:
        if self._values is None:
            v = np.unpackbits(self.bits, count=self.grid.n_pts).reshape(self.grid.dims)
            v.setflags(write=False)
            self._values = v
        return self._values

    def solid_count(self) -> int:
        return int(np.bitwise_count(self.bits).sum())

    def solid_fraction(self) -> float:
        return self.solid_count() / self.grid.n_pts

    def all_solid(self) -> bool:
        return self.solid_count() == self.grid.n_pts

    @property
    def degenerate(self) -> bool:
        frac = self.solid_fraction()
        return frac == 0.0 or frac == 1.0

    def as_float(self) -> np.ndarray:
        return self.values.astype(np.float64)


def all_solid(indicator) -> bool:
    """True if every voxel is solid (the solvers' fast path); packed indicators
    answer from a popcount of their bits."""
    f = getattr(indicator, "all_solid", None)
    return bool(f()) if f is not None else bool(np.asarray(indicator.values).all())


def porosity(indicator: IndicatorField) -> float:
    """grid.py:108-110."""
    return 1.0 - indicator.solid_fraction()


def make_model_geometry(grid: UnitCellGrid, radius: float = 0.25, center=None) -> IndicatorField:
    """Centred ball (disk in 2D) of the given radius.  grid.py:113-131."""
    if not 0.0 < radius < 0.5:
        raise ValueError(f"obstacle radius must be in (0, 0.5), got {radius}")
    if center is None:
        center = (0.5,) * grid.dim
    if len(center) != grid.dim:
        raise ValueError("center must have one coordinate per grid axis")
    coords = grid.meshgrid()
    r_sq = sum((y - c) ** 2 for y, c in zip(coords, center))
    return IndicatorField(grid, (r_sq <= radius ** 2).astype(np.uint8))


@dataclass(frozen=True)
class SpherePacking:
    """Sphere centres (unit-cell coordinates) and radii of a periodic packing."""

    centers: np.ndarray
    radii: np.ndarray

    @property
    def solid_fraction(self) -> float:
        return float((4.0 / 3.0) * np.pi * np.sum(self.radii ** 3))


def random_sphere_packing(seed: int = 0, r_min: float = 0.04, r_max: float = 0.08,
                          target_solid_fraction: float = 0.30, max_attempts: int = 200_000) -> SpherePacking:
    """Periodic random sequential addition of non-overlapping spheres.

    SURVEY.md §8d cfg 3: radii ~ U[r_min, r_max] (unit-cell lengths), centres
    ~ U[0,1)^3 from ``np.random.default_rng(seed)``; a candidate is accepted
    when its minimum-image distance to every accepted sphere is at least the
    sum of radii; stops once the analytic solid fraction reaches the target.
    Resolution independent: rasterise with ``rasterize_packing``.
    """
    rng = np.random.default_rng(seed)
    centers = np.zeros((0, 3))
    radii = np.zeros(0)
    vol = 0.0
    attempts = 0
    while vol < target_solid_fraction:
        if attempts >= max_attempts:
            raise RuntimeError("random sequential addition jammed before the target fraction")
        attempts += 1
        r = rng.uniform(r_min, r_max)
        c = rng.random(3)
        if radii.size:
            dv = centers - c
            dv -= np.round(dv)
            if np.any(np.einsum("ij,ij->i", dv, dv) < (radii + r) ** 2):
                continue
        centers = np.vstack([centers, c])
        radii = np.append(radii, r)
        vol += (4.0 / 3.0) * np.pi * r ** 3
    return SpherePacking(centers, radii)


def rasterize_packing(packing: SpherePacking, dims) -> IndicatorField:
    """Indicator at cell centres, minimum-image criterion d^2 <= r^2 (grid.py:129-131)."""
    grid = UnitCellGrid(tuple(dims))
    if grid.dim != 3:
        raise ValueError("sphere packings are 3D")
    solid = np.zeros(grid.dims, dtype=bool)
    for c, r in zip(packing.centers, packing.radii):
        sel, d2 = [], []
        for a in range(3):
            n = grid.dims[a]
            lo = int(np.floor((c[a] - r) * n - 0.5)) - 1
            hi = int(np.ceil((c[a] + r) * n - 0.5)) + 1
            idx = np.arange(lo, hi + 1)
            y = (idx + 0.5) / n
            dy = y - c[a]
            dy -= np.round(dy)
            keep = dy * dy <= r * r
            sel.append(np.mod(idx[keep], n))
            d2.append(dy[keep] ** 2)
        if any(s.size == 0 for s in sel):
            continue
        inside = (d2[0][:, None, None] + d2[1][None, :, None] + d2[2][None, None, :]) <= r * r
        ix = np.ix_(*sel)
        solid[ix] |= inside
    return IndicatorField(grid, solid.astype(np.uint8))


def random_packing_geometry(n: int, seed: int = 0, **kwargs) -> IndicatorField:
    """BASELINE cfg-3/4/5 microstructure at n^3."""
    return rasterize_packing(random_sphere_packing(seed, **kwargs), (n, n, n))


def rasterize_packing_slab(packing: SpherePacking, dims, lo: int, hi: int) -> np.ndarray:
    """The x-slab i0 in [lo, hi) of ``rasterize_packing(packing, dims).values``
    (uint8, (hi - lo, N1, N2)) without materialising the whole cell — each rank
    of a slab-decomposed solve (slab.py) builds only its own planes."""
    dims = tuple(int(x) for x in dims)
    if len(dims) != 3 or not (0 <= lo < hi <= dims[0]):
        raise ValueError("slab rasterization needs 3D dims and 0 <= lo < hi <= N0")
    solid = np.zeros((hi - lo,) + dims[1:], dtype=bool)
    for c, r in zip(packing.centers, packing.radii):
        sel, d2 = [], []
        for a in range(3):
            n = dims[a]
            a_lo = int(np.floor((c[a] - r) * n - 0.5)) - 1
            a_hi = int(np.ceil((c[a] + r) * n - 0.5)) + 1
            idx = np.arange(a_lo, a_hi + 1)
            y = (idx + 0.5) / n
            dy = y - c[a]
            dy -= np.round(dy)
            keep = dy * dy <= r * r
            ii = np.mod(idx[keep], n)
            dd = dy[keep] ** 2
            if a == 0:  # only this slab's planes, shifted to local indices
                m = (ii >= lo) & (ii < hi)
                ii, dd = ii[m] - lo, dd[m]
            sel.append(ii)
            d2.append(dd)
        if any(x.size == 0 for x in sel):
            continue
        inside = (d2[0][:, None, None] + d2[1][None, :, None] + d2[2][None, None, :]) <= r * r
        solid[np.ix_(*sel)] |= inside
    return solid.astype(np.uint8)
