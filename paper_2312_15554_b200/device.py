"""Device plumbing: CUDA device selection, plan cache, host<->device moves.

PyTorch supplies device memory and the current stream; the compute is the
native library.  One ``Plan`` per (grid, symbol mode, device, host thread):
plans are not thread-safe, mirroring the reference's "independent solver
instances" contract (tests/test_backends.py:131-149).
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

from . import _native as N

_SYMBOL_CODES = {"exact": N.PF_SYMBOLS_EXACT, "central": N.PF_SYMBOLS_CENTRAL}


def torch():
    import torch as _t

    return _t


def require_cuda(device=None):
    """The CUDA device to use; raises when none is available (no CPU fallback)."""
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("poreflow_b200 needs a CUDA device (B200, sm_100a); none is visible")
    N.load()
    if device is None:
        return t.device("cuda", t.cuda.current_device())
    dev = t.device(device)
    if dev.type != "cuda":
        raise ValueError(f"poreflow_b200 computes on CUDA devices only, got {dev}")
    return t.device("cuda", dev.index if dev.index is not None else t.cuda.current_device())


class Plan:
    """Owns one ``pf_plan*``: grid geometry, symbol tables, cuFFT plans, scratch."""

    def __init__(self, dims, mode: str, device):
        from .spectral import symbol_tables

        t = torch()
        self.dims = tuple(int(n) for n in dims)
        self.mode = mode
        self.device = device
        lib = N.load()
        h = ctypes.c_void_p()
        with t.cuda.device(device):
            stream = t.cuda.current_stream(device).cuda_stream
            N.check(lib.pf_plan_create(ctypes.byref(h), len(self.dims), N.i64_array(self.dims),
                                       _SYMBOL_CODES[mode], device.index, ctypes.c_void_p(stream)))
        self.handle = h
        # numpy's own tables, so the device uses the reference's bits (spectral.py:78-86)
        for ax, (kap, lap1) in enumerate(symbol_tables(self.dims, mode)):
            kap = np.ascontiguousarray(kap, dtype=np.float64)
            lap1 = np.ascontiguousarray(lap1, dtype=np.float64)
            N.check(lib.pf_plan_set_symbol_tables(h, ax, kap.ctypes.data, lap1.ctypes.data))

    def bind_stream(self):
        t = torch()
        stream = t.cuda.current_stream(self.device).cuda_stream
        N.check(N.load().pf_plan_set_stream(self.handle, ctypes.c_void_p(stream)))
        return self.handle

    def device_bytes(self) -> int:
        out = ctypes.c_size_t()
        N.check(N.load().pf_plan_device_bytes(self.handle, ctypes.byref(out)))
        return int(out.value)

    def close(self):
        if getattr(self, "handle", None):
            N.load().pf_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_plans = threading.local()


def get_plan(dims, mode: str, device=None, slot: int = 0) -> Plan:
    """Cached plan for (grid, symbol mode, device, slot) on this host thread.

    Concurrent solves (one CUDA stream each, e.g. an ensemble of cells on one
    GPU) need distinct ``slot`` values: a plan owns its scratch and stream."""
    device = require_cuda(device)
    cache = getattr(_plans, "cache", None)
    if cache is None:
        cache = _plans.cache = {}
    key = (tuple(int(n) for n in dims), mode, device.index, int(slot))
    plan = cache.get(key)
    if plan is None:
        plan = cache[key] = Plan(dims, mode, device)
    return plan


def release_plans() -> None:
    """Free every plan (and its device scratch) owned by this host thread."""
    cache = getattr(_plans, "cache", None) or {}
    for p in cache.values():
        p.close()
    cache.clear()


def to_device(arr, device, dtype=None):
    """numpy array / torch tensor -> contiguous CUDA tensor (copy for numpy)."""
    t = torch()
    if isinstance(arr, t.Tensor):
        x = arr.to(device=device, dtype=dtype or arr.dtype)
        return x.contiguous()
    a = np.ascontiguousarray(arr, dtype=dtype and _np_dtype(dtype))
    if not a.flags.writeable:
        a = a.copy()
    return t.from_numpy(a).to(device=device, non_blocking=False)


def solid_on_device(indicator, device):
    """Device copy of an (immutable) indicator's uint8 values, cached on this
    package's IndicatorField; duck-typed indicators (e.g. the reference's own
    ``poreflow.IndicatorField``) are copied per call."""
    cache = getattr(indicator, "_device_cache", None)
    if cache is None:
        return to_device(np.asarray(indicator.values, dtype=np.uint8), device, torch().uint8)
    key = device.index
    if key not in cache:
        bits = getattr(indicator, "bits", None)
        cache[key] = (_unpack_on_device(bits, indicator.grid.n_pts, device).reshape(indicator.grid.dims)
                      if bits is not None else to_device(indicator.values, device, torch().uint8))
    return cache[key]


def _unpack_on_device(bits, n: int, device):
    """Packed indicator bytes -> device uint8 0/1 per voxel (pf_unpack_bits)."""
    t = torch()
    dbits = to_device(np.asarray(bits, dtype=np.uint8), device, t.uint8)
    out = t.empty(n, dtype=t.uint8, device=device)
    with t.cuda.device(device):
        stream = t.cuda.current_stream(device).cuda_stream
        N.check(N.load().pf_unpack_bits(ctypes.c_void_p(dbits.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                        int(n), ctypes.c_void_p(stream)))
    return out


_STAGE_BYTES = 16 << 20
_STAGES = max(4, min(8, os.cpu_count() or 4))
_stage = threading.local()


def _stage_buffers():
    st = getattr(_stage, "bufs", None)
    if st is None:
        t = torch()
        _stage.bufs = [t.empty(_STAGE_BYTES, dtype=t.uint8, pin_memory=True) for _ in range(_STAGES)]
        _stage.events = [t.cuda.Event() for _ in range(_STAGES)]
        from concurrent.futures import ThreadPoolExecutor

        _stage.pool = ThreadPoolExecutor(max_workers=_STAGES)
    return _stage.bufs, _stage.events, _stage.pool


_NP = None


def _np_dtype(dt):
    global _NP
    if _NP is None:
        t = torch()
        _NP = {t.float64: np.float64, t.uint8: np.uint8, t.complex128: np.complex128, t.float32: np.float32}
    return _NP[dt]


# Results up to this many bytes per call come back in pinned host memory: one direct
# DMA per field at full PCIe rate, with the blocks recycled by torch's caching host
# allocator once the caller drops the arrays.  Larger states (or 0 here) use the
# staged ring below, whose output is ordinary pageable memory.
_PINNED_OUT_BYTES = int(float(os.environ.get("POREFLOW_B200_PINNED_OUT_GB", "8")) * (1 << 30))

# A dropped result's pinned blocks go back to torch's caching host allocator and are
# reused by the next result, but blocks still held by live results cannot be:
# pinning fresh memory costs ~0.6 s per GB (page locking), several times what the
# staged ring needs for the whole copy.  So after the first large result, a large
# result comes back pinned only when at least as many pinned result bytes have been
# released since (the caller dropped earlier results); otherwise through the ring.
# (A caller that keeps every load case's state pays the page locking once, not per
# solve; a loop that drops each state before the next keeps the direct DMA path.)
_pin_lock = threading.Lock()
_pin_state = {"used": False, "released": 0}


def _pinned_ok(total: int) -> bool:
    if total <= (64 << 20):
        return True
    with _pin_lock:
        if not _pin_state["used"]:
            _pin_state["used"] = True
            return True
        if _pin_state["released"] >= total:
            _pin_state["released"] -= total
            return True
        return False


def _pinned_released(nbytes: int) -> None:
    with _pin_lock:
        _pin_state["released"] += nbytes


def to_host_many(xs) -> list:
    """CUDA tensors -> new numpy arrays.

    Small results (see ``_PINNED_OUT_BYTES``): arrays backed by pinned host memory,
    filled by direct device-to-host copies.  Otherwise ONE pipeline: device-to-host DMA
    into a ring of pinned staging buffers (~55 GB/s) overlapped with parallel host
    copies out of them (numpy releases the GIL).  The host side is bound by
    first-touch page faults of the fresh output arrays (~4 GB/s per thread), so
    the ring is as wide as the host has threads and runs across all fields
    instead of draining per field."""
    t = torch()
    xs = [x.contiguous() for x in xs]
    total = sum(x.numel() * x.element_size() for x in xs)
    if total <= _PINNED_OUT_BYTES and _pinned_ok(total):
        hs = [t.empty(tuple(x.shape), dtype=x.dtype, pin_memory=True) for x in xs]
        for h, x in zip(hs, xs):
            h.copy_(x, non_blocking=True)
        if xs:
            t.cuda.current_stream(xs[0].device).synchronize()
        outs = [h.numpy() for h in hs]
        if total > (64 << 20):  # (the array, and every view of it, holds the pinned block)
            for o in outs:
                weakref.finalize(o, _pinned_released, o.nbytes)
        return outs
    outs = [np.empty(tuple(x.shape), dtype=_np_dtype(x.dtype)) for x in xs]
    big = [i for i, o in enumerate(outs) if o.nbytes > (4 << 20)]
    for i, o in enumerate(outs):
        if i not in big:
            o[...] = xs[i].cpu().numpy()
    if not big:
        return outs
    bufs, evs, pool = _stage_buffers()
    chunks = []
    for i in big:
        nb = outs[i].nbytes
        chunks += [(i, o, min(_STAGE_BYTES, nb - o)) for o in range(0, nb, _STAGE_BYTES)]
    srcs = {i: xs[i].view(-1).view(t.uint8) for i in big}
    dsts = {i: outs[i].reshape(-1).view(np.uint8) for i in big}
    pending = [None] * _STAGES

    def host_copy(j, i, o, k):
        evs[j].synchronize()
        np.copyto(dsts[i][o:o + k], bufs[j][:k].numpy())

    for n, (i, o, k) in enumerate(chunks):
        j = n % _STAGES
        if pending[j] is not None:
            pending[j].result()  # staging buffer j is free again
        bufs[j][:k].copy_(srcs[i][o:o + k], non_blocking=True)
        evs[j].record(t.cuda.current_stream(xs[i].device))
        pending[j] = pool.submit(host_copy, j, i, o, k)
    for f in pending:
        if f is not None:
            f.result()
    return outs


def to_host(x) -> np.ndarray:
    """CUDA tensor -> new numpy array (see ``to_host_many``)."""
    return to_host_many([x])[0]
