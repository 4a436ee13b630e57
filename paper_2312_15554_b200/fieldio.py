"""Field, history, report and raster I/O — the reference's interchange formats
(pkg/src/poreflow/fieldio.py, grid.py:135-217) so a run here writes files the
reference's readers and viewers accept, plus the 3D formats the reference lacks.

Kept byte-compatible with the reference (2D):
  * field CSV: one file per component, header ``poreflow-field v1`` / dims /
    spacing / component, data rows along the second grid axis, ``%.17g``
    (fieldio.py:56-68);
  * legacy ASCII VTK STRUCTURED_POINTS, first axis fastest (fieldio.py:89-112);
  * residual-history CSV (fieldio.py:115-125) and report JSON, indent 2, sorted
    keys, numpy arrays as lists (fieldio.py:128-140);
  * indicator rasters: binary PGM (P5) and integer CSV, file rows along the
    second axis, solid where value >= threshold (grid.py:135-217).

New for 3D (the reference's VTK and rasters are 2D-only):
  * VTK STRUCTURED_POINTS of any dimension (x fastest);
  * ``.npy`` fields and indicators of any dimension;
  * raw voxel files (``load_indicator_raw``: uint8 / float, C order, given dims).

Host-side file formats only; nothing here touches the device.
"""

from __future__ import annotations

import json
import re
from pathlib import Path

import numpy as np

from .grid import IndicatorField, PackedIndicator, UnitCellGrid
from .report import ConvergenceReport

_FMT = "%.17g"
FIELD_HEADER = "poreflow-field v1"
_PGM_MAXVAL = 255


def _component_views(field: np.ndarray, grid: UnitCellGrid):
    if field.shape == grid.dims:
        return [field]
    if field.ndim == grid.dim + 1 and field.shape[1:] == grid.dims:
        return [field[c] for c in range(field.shape[0])]
    raise ValueError(f"field shape {field.shape} does not match grid {grid.dims}")


def export_field(field, grid: UnitCellGrid, fmt: str, path, name: str = "field") -> list[Path]:
    """Write a scalar or vector field; returns the paths written (fieldio.py:31-53).

    ``csv``: 2D grids, one file per component suffixed ``_c0``, ``_c1``, ...;
    ``vtk``: all components in one legacy file (2D as the reference, 3D new);
    ``npy``: the array as is, any dimension (new)."""
    field = np.asarray(field)
    path = Path(path)
    if fmt == "csv":
        if grid.dim != 2:
            raise ValueError("CSV field export is defined for 2D grids (use 'vtk' or 'npy' in 3D)")
        comps = _component_views(field, grid)
        paths = []
        for c, comp in enumerate(comps):
            p = path if len(comps) == 1 else path.with_name(f"{path.stem}_c{c}{path.suffix}")
            _write_csv_component(comp, grid, p, component=c, n_components=len(comps))
            paths.append(p)
        return paths
    if fmt == "vtk":
        _write_vtk(field, grid, path, name)
        return [path]
    if fmt == "npy":
        _component_views(field, grid)  # shape check
        np.save(path, field)
        return [path]
    raise ValueError(f"unknown field format {fmt!r} (expected 'csv', 'vtk' or 'npy')")


def _write_csv_component(comp, grid, path, component, n_components):
    spacing = ",".join(_FMT % h for h in grid.spacing)
    dims = ",".join(str(n) for n in grid.dims)
    header = f"{FIELD_HEADER}\ndims: {dims}\nspacing: {spacing}\ncomponent: {component}/{n_components}"
    np.savetxt(path, comp.T, fmt=_FMT, delimiter=",", header=header)


def import_field_csv(path) -> tuple[np.ndarray, UnitCellGrid]:
    """Read one CSV component back; inverse of the CSV writer (fieldio.py:71-86)."""
    path = Path(path)
    dims = None
    with open(path) as fh:
        for line in fh:
            if not line.startswith("#"):
                break
            if line[1:].strip().startswith("dims:"):
                dims = tuple(int(t) for t in line.split(":")[1].split(","))
    data = np.loadtxt(path, delimiter=",", ndmin=2).T
    grid = UnitCellGrid(dims if dims is not None else data.shape)
    if data.shape != grid.dims:
        raise ValueError(f"data shape {data.shape} does not match header dims {dims}")
    return data, grid


def _write_vtk(field, grid, path, name):
    comps = _component_views(field, grid)
    d = grid.dim
    if d not in (2, 3):
        raise ValueError("VTK export is defined for 2D and 3D grids")
    n = list(grid.dims) + [1] * (3 - d)
    h = list(grid.spacing) + [1] * (3 - d)
    origin = [0.5 * x for x in grid.spacing] + [0] * (3 - d)
    fmt_o = lambda v: _FMT % v if isinstance(v, float) else str(v)  # noqa: E731
    lines = [
        "# vtk DataFile Version 3.0",
        f"poreflow field {name}",
        "ASCII",
        "DATASET STRUCTURED_POINTS",
        "DIMENSIONS " + " ".join(str(k) for k in n),
        "ORIGIN " + " ".join(fmt_o(v) for v in origin),
        "SPACING " + " ".join(fmt_o(v) for v in h),
        f"POINT_DATA {grid.n_pts}",
    ]
    for c, comp in enumerate(comps):
        label = name if len(comps) == 1 else f"{name}_{c + 1}"
        lines.append(f"SCALARS {label} double 1")
        lines.append("LOOKUP_TABLE default")
        # structured points run x fastest: reverse the axis order of the C-order array
        lines.extend(_FMT % v for v in np.transpose(comp).ravel())
    Path(path).write_text("\n".join(lines) + "\n")


def write_history_csv(report: ConvergenceReport, path) -> Path:
    """Residual history, one row per iteration (fieldio.py:115-125)."""
    path = Path(path)
    np.savetxt(path, report.history, fmt=_FMT, delimiter=",", header="iteration history: " + ",".join(report.columns))
    return path


def read_history_csv(path) -> ConvergenceReport:
    """Inverse of ``write_history_csv`` (columns from the header; flags unknown)."""
    path = Path(path)
    with open(path) as fh:
        head = fh.readline()
    cols = tuple(head.split(":", 1)[1].strip().split(","))
    hist = np.loadtxt(path, delimiter=",", ndmin=2)
    return ConvergenceReport(cols, hist, converged=False, iterations=hist.shape[0])


class _NumpyEncoder(json.JSONEncoder):
    def default(self, obj):
        if isinstance(obj, np.ndarray):
            return obj.tolist()
        if isinstance(obj, (np.floating, np.integer)):
            return obj.item()
        return super().default(obj)


def write_report_json(report: dict, path) -> Path:
    """Report as JSON, indent 2, sorted keys (fieldio.py:137-140)."""
    path = Path(path)
    path.write_text(json.dumps(report, indent=2, sort_keys=True, cls=_NumpyEncoder) + "\n")
    return path


# ---------------------------------------------------------------------------
# Indicator rasters (grid.py:135-217) and 3D voxel ingest.

def load_indicator_raster(path, threshold: float = 0.5) -> IndicatorField:
    """Indicator from a raster file: solid where value >= threshold.

    ``.pgm`` (binary P5, normalised by maxval) and CSV (anything else, values as
    is) are the reference's 2D formats (grid.py:135-160): the file's rows run
    along the second grid axis.  ``.npy`` holds an array of any dimension in grid
    order (C order, first axis slowest), compared as is."""
    path = Path(path)
    if not path.exists():
        raise FileNotFoundError(path)
    suffix = path.suffix.lower()
    if suffix == ".npy":
        vals = np.load(path)
        if vals.size == 0:
            raise ValueError(f"empty raster: {path}")
        values = (vals >= threshold).astype(np.uint8)
        return IndicatorField(UnitCellGrid(values.shape), values)
    pixels = _read_pgm(path) / _PGM_MAXVAL if suffix == ".pgm" else _read_csv_raster(path)
    if pixels.size == 0:
        raise ValueError(f"empty raster: {path}")
    values = (pixels.T >= threshold).astype(np.uint8)  # file rows run along the second grid axis
    return IndicatorField(UnitCellGrid(values.shape), values)


def load_indicator_raw(path, dims, dtype=np.uint8, threshold: float = 0.5) -> IndicatorField:
    """3D (any-D) raw voxel file: ``prod(dims)`` values of ``dtype``, C order."""
    path = Path(path)
    if not path.exists():
        raise FileNotFoundError(path)
    dims = tuple(int(n) for n in dims)
    vals = np.fromfile(path, dtype=dtype)
    if vals.size != int(np.prod(dims)):
        raise ValueError(f"raw file holds {vals.size} values, dims {dims} need {int(np.prod(dims))}: {path}")
    values = (vals.reshape(dims) >= threshold).astype(np.uint8)
    return IndicatorField(UnitCellGrid(dims), values)


def load_indicator_bits(path, dims) -> PackedIndicator:
    """Bit-packed voxel file (numpy.packbits order, C order, ceil(prod(dims) / 8)
    bytes): stays packed on the host; the device solvers unpack it on the GPU."""
    path = Path(path)
    if not path.exists():
        raise FileNotFoundError(path)
    return PackedIndicator(UnitCellGrid(tuple(int(n) for n in dims)), np.fromfile(path, dtype=np.uint8))


def save_indicator_bits(indicator, path) -> Path:
    """Write an indicator as a bit-packed voxel file (see ``load_indicator_bits``)."""
    path = Path(path)
    bits = getattr(indicator, "bits", None)
    if bits is None:
        bits = np.packbits(np.asarray(indicator.values, dtype=np.uint8).ravel())
    np.asarray(bits, dtype=np.uint8).tofile(path)
    return path


def write_indicator(indicator: IndicatorField, path) -> Path:
    """PGM (``.pgm``) or CSV (other suffixes) for 2D, as the reference
    (grid.py:163-173); ``.npy`` for any dimension."""
    path = Path(path)
    values = np.asarray(indicator.values)
    if path.suffix.lower() == ".npy":
        np.save(path, values.astype(np.uint8))
        return path
    if indicator.grid.dim != 2:
        raise ValueError("raster output is defined for 2D indicators (use .npy in 3D)")
    raster = values.T  # file rows = second axis
    if path.suffix.lower() == ".pgm":
        _write_pgm(path, (raster * _PGM_MAXVAL).astype(np.uint8))
    else:
        np.savetxt(path, raster, fmt="%d", delimiter=",")
    return path


def _read_pgm(path: Path) -> np.ndarray:
    data = path.read_bytes()
    tokens, pos = [], 0
    while len(tokens) < 4:  # magic, width, height, maxval; '#' comments allowed between tokens
        m = re.match(rb"\s*(?:#[^\n]*\n\s*)*(\S+)", data[pos:])
        if m is None:
            raise ValueError(f"truncated PGM header: {path}")
        tokens.append(m.group(1))
        pos += m.end()
    if tokens[0] != b"P5":
        raise ValueError(f"not a binary PGM (P5) file: {path}")
    width, height, maxval = (int(t) for t in tokens[1:])
    if maxval <= 0 or maxval > _PGM_MAXVAL:
        raise ValueError(f"unsupported PGM maxval {maxval}: {path}")
    pos += 1  # one whitespace byte separates header and pixels
    if len(data) < pos + width * height:
        raise ValueError(f"PGM pixel data shorter than header promises: {path}")
    pixels = np.frombuffer(data, dtype=np.uint8, count=width * height, offset=pos)
    return pixels.reshape(height, width).astype(np.float64) * (_PGM_MAXVAL / maxval)


def _write_pgm(path: Path, raster: np.ndarray) -> None:
    height, width = raster.shape
    with open(path, "wb") as fh:
        fh.write(f"P5\n{width} {height}\n{_PGM_MAXVAL}\n".encode())
        fh.write(raster.tobytes())


def _read_csv_raster(path: Path) -> np.ndarray:
    try:
        return np.loadtxt(path, delimiter=",", ndmin=2)
    except ValueError as exc:
        raise ValueError(f"non-rectangular or malformed CSV raster: {path}") from exc
