"""Slab-decomposed Stokes solve of ONE cell across ranks (BASELINE cfg 5).

Rank r holds the x-slab i0 in [r N0/P, (r+1) N0/P) of every real field and the
y-slab k1 in [r N1/P, ...) of every spectrum.  Per ADMM iteration the ranks
exchange two half spectra (R^ forward, U^ back, 3 components each) with
``all_to_all`` and all-reduce the 9 squared-norm partial sums; every decision
(residuals, convergence, residual balancing — stokes.py:247-310) then runs on
identical totals on every rank, so all ranks stop at the same iteration.

The driver is backend-agnostic: ``DeviceSlabBackend`` runs the per-rank work on
the GPU through ``pf_slab_*`` (include/poreflow_b200.h) and the collectives go
through ``torch.distributed`` (NCCL on the GPU box); the CPU tests drive the
same loop with a numpy test double over ``gloo``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .device import require_cuda, torch
from .report import ConvergenceReport
from .spectral import CENTRAL as CENTRAL_MODE
from .stokes import REPORT_COLUMNS, PenaltyParams, StokesConfig, _params


def slab_range(n0: int, world: int, rank: int) -> tuple[int, int]:
    """x-slab [lo, hi) of rank ``rank`` (N0 must be divisible by the world size)."""
    if n0 % world:
        raise ValueError(f"N0 = {n0} is not divisible by {world} ranks")
    L0 = n0 // world
    return rank * L0, (rank + 1) * L0


class DeviceSlabBackend:
    """Per-rank device work through the C ABI; buffers are CUDA tensors."""

    def __init__(self, dims, world: int, rank: int, symbol_mode: str = "central", device=None):
        from .device import _SYMBOL_CODES
        from .spectral import symbol_tables

        self.dev = require_cuda(device)
        t = torch()
        lib = N.load()
        h = ctypes.c_void_p()
        with t.cuda.device(self.dev):
            stream = t.cuda.current_stream(self.dev).cuda_stream
            N.check(lib.pf_slab_plan_create(ctypes.byref(h), N.i64_array(dims), world, rank,
                                            _SYMBOL_CODES[symbol_mode], self.dev.index, ctypes.c_void_p(stream)))
        self.h = h
        for ax, (kap, lap1) in enumerate(symbol_tables(tuple(dims), symbol_mode)):
            kap = np.ascontiguousarray(kap, dtype=np.float64)
            lap1 = np.ascontiguousarray(lap1, dtype=np.float64)
            N.check(lib.pf_plan_set_symbol_tables(h, ax, kap.ctypes.data, lap1.ctypes.data))
        e, ts, r = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        N.check(lib.pf_slab_sizes(h, ctypes.byref(e), ctypes.byref(ts), ctypes.byref(r)))
        self.exch, self.tspec, self.real = int(e.value), int(ts.value), int(r.value)
        self.lib = lib

    def _p(self, x):
        return ctypes.c_void_p(x.data_ptr())

    def bind(self):
        t = torch()
        N.check(self.lib.pf_plan_set_stream(self.h, ctypes.c_void_p(t.cuda.current_stream(self.dev).cuda_stream)))

    # buffers: complex buffers are float64 tensors holding interleaved (re, im)
    def alloc_complex(self, count):
        t = torch()
        return t.empty(2 * count, dtype=t.float64, device=self.dev)

    def alloc_real(self, count):
        t = torch()
        return t.empty(count, dtype=t.float64, device=self.dev)

    def forward(self, real, ncomp, send):
        N.check(self.lib.pf_slab_forward(self.h, self._p(real), ncomp, self._p(send)))

    def forward_finish(self, recv, ncomp, tspec):
        N.check(self.lib.pf_slab_forward_finish(self.h, self._p(recv), ncomp, self._p(tspec)))

    def inverse(self, tspec, ncomp, send):
        N.check(self.lib.pf_slab_inverse(self.h, self._p(tspec), ncomp, self._p(send)))

    def inverse_finish(self, recv, ncomp, real):
        N.check(self.lib.pf_slab_inverse_finish(self.h, self._p(recv), ncomp, self._p(real)))

    def begin(self, params, solid, u, ut, q, a, lam, hist):
        N.check(self.lib.pf_slab_stokes_begin(self.h, ctypes.byref(params), self._p(solid), self._p(u), self._p(ut),
                                              self._p(q), self._p(a), self._p(lam), self._p(hist)))

    def setup(self, Tq, Tu, Q, D):
        N.check(self.lib.pf_slab_setup(self.h, self._p(Tq), self._p(Tu), self._p(Q), self._p(D)))

    def spectral(self, R, Q, D, U):
        N.check(self.lib.pf_slab_spectral(self.h, self._p(R), self._p(Q), self._p(D), self._p(U)))

    def local(self, unew, totals):
        N.check(self.lib.pf_slab_local(self.h, self._p(unew), self._p(totals)))

    def finalize(self, totals):
        N.check(self.lib.pf_slab_finalize(self.h, self._p(totals)))

    def form_r(self, R, gated):
        N.check(self.lib.pf_slab_form_r(self.h, self._p(R), 1 if gated else 0))

    def scale(self, src, dst, count, s):
        N.check(self.lib.pf_slab_scale(self.h, self._p(src), self._p(dst), int(count), float(s)))

    def grad(self, tspec, axis, out):
        N.check(self.lib.pf_slab_grad(self.h, self._p(tspec), int(axis), self._p(out)))

    def gram(self, solid, G) -> np.ndarray:
        out = (ctypes.c_double * 6)()
        N.check(self.lib.pf_slab_gram(self.h, self._p(solid), self._p(G), out))
        return np.asarray(out[:])

    # fused slab pipeline (pf_slab_fused_*)
    def fused_sizes(self) -> tuple:
        m, q = ctypes.c_int64(), ctypes.c_int64()
        N.check(self.lib.pf_slab_fused_sizes(self.h, ctypes.byref(m), ctypes.byref(q)))
        return int(m.value), int(q.value)

    def fused_bind(self, Yy, Yyn, Yx, Yxn):
        N.check(self.lib.pf_slab_fused_bind(self.h, self._p(Yy), self._p(Yyn), self._p(Yx), self._p(Yxn)))

    def fused_setup(self, Q, D, R):
        N.check(self.lib.pf_slab_fused_setup(self.h, self._p(Q), self._p(D), self._p(R)))

    def fused_setup_zero(self):
        N.check(self.lib.pf_slab_fused_setup_zero(self.h))

    def release_transforms(self):
        N.check(self.lib.pf_slab_release_transforms(self.h))

    def fused_pk(self):
        N.check(self.lib.pf_slab_fused_pk(self.h))

    def fused_rs(self, totals):
        N.check(self.lib.pf_slab_fused_rs(self.h, self._p(totals)))

    def fused_mf(self):
        N.check(self.lib.pf_slab_fused_mf(self.h))

    def fused_rs_part(self, comp):
        N.check(self.lib.pf_slab_fused_rs_part(self.h, int(comp)))

    def fused_totals(self, totals):
        N.check(self.lib.pf_slab_fused_totals(self.h, self._p(totals)))

    def fused_mf_part(self, comp, fix):
        N.check(self.lib.pf_slab_fused_mf_part(self.h, int(comp), 1 if fix else 0))

    def fused_set_peers(self, yy, yyn, yx, yxn):
        """Peer-memory exchange: lists (rank order) of every rank's Y buffer
        addresses, mapped in this process; empty lists restore all_to_all."""
        arr = lambda v: (ctypes.c_uint64 * max(1, len(v)))(*[int(x) for x in v])  # noqa: E731
        N.check(self.lib.pf_slab_fused_set_peers(self.h, arr(yy), arr(yyn), arr(yx), arr(yxn), len(yy)))

    def fused_end(self, Q):
        N.check(self.lib.pf_slab_fused_end(self.h, self._p(Q)))

    def read(self) -> dict:
        r = N.StokesResult()
        N.check(self.lib.pf_slab_read(self.h, ctypes.byref(r)))
        return {"iterations": int(r.iterations), "converged": bool(r.converged), "done": bool(r.done),
                "final_penalties": tuple(float(x) for x in r.final_penalties)}

    def close(self):
        if self.h:
            self.lib.pf_plan_destroy(self.h)
            self.h = None


class SlabStokes:
    """ADMM Stokes loop (stokes.py:313-427) over a slab-decomposed cell.

    ``state`` = dict of the rank's local fields u, u_tilde, a, lam (3, L0, N1, N2)
    and q (L0, N1, N2) as backend tensors (flattened), updated in place.
    """

    def __init__(self, backend, dims, cfg: StokesConfig, penalties: PenaltyParams | None, solid_local, state,
                 group=None, poll_every: int = 8, comm=None, overlap: bool = True):
        """``comm``: an object with torch.distributed's ``get_world_size`` /
        ``all_to_all_single`` / ``all_reduce`` (default: torch.distributed when
        initialised); tests inject an in-process loopback to run P ranks on one GPU.
        ``overlap``: pipeline every 3-component exchange per component (async
        all_to_all) so component c's transfer overlaps the local
        transforms of its neighbours; False = one blocking exchange per transform."""
        import torch.distributed as dist

        self.b, self.dims, self.cfg = backend, tuple(int(x) for x in dims), cfg
        self.pen = penalties or PenaltyParams()
        self.solid, self.state, self.group, self.poll = solid_local, state, group, max(1, int(poll_every))
        self.overlap = bool(overlap)
        if comm is not None:
            self.dist = comm
        else:
            self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.world = self.dist.get_world_size(group) if self.dist else 1
        be = backend
        if self._eager_buffers:
            self._alloc_buffers(3)
        self.totals = be.alloc_real(9)
        self.hist = be.alloc_real(cfg.max_iter * len(REPORT_COLUMNS))

    # the cuFFT-slab transform buffers (every iteration of SlabStokes; only setup
    # and teardown of FusedSlabStokes, which allocates them for those phases only)
    _eager_buffers = True

    def _alloc_buffers(self, ncomp, teardown: bool = False):
        """``teardown``: only what end() needs (Q^, one T-layout component, one
        component's exchange buffers)."""
        be = self.b
        self.send = be.alloc_complex(ncomp * be.exch)
        self.recv = be.alloc_complex(ncomp * be.exch) if self.world > 1 else self.send
        self.TU = be.alloc_complex(ncomp * be.tspec)
        self.Q = be.alloc_complex(be.tspec)
        if teardown:
            return
        self.TR = be.alloc_complex(ncomp * be.tspec)
        self.D = be.alloc_complex(be.tspec)
        self.R = be.alloc_real(ncomp * be.real)
        self.unew = be.alloc_real(ncomp * be.real)

    def _free_buffers(self):
        self.send = self.recv = self.TR = self.TU = self.Q = self.D = self.R = self.unew = None

    def _exchange(self, ncomp):
        if self.world == 1:
            return
        k = 2 * ncomp * self.b.exch
        self.dist.all_to_all_single(self.recv[:k], self.send[:k], group=self.group)

    def _a2a(self, out, inp):
        """Asynchronous all_to_all of equal contiguous splits; the returned handle's
        ``wait()`` orders the caller's stream after it (NCCL) or blocks (gloo)."""
        return self.dist.all_to_all_single(out, inp, group=self.group, async_op=True)

    def _pipelined(self, ncomp):
        return self.overlap and self.world > 1 and ncomp > 1

    def _to_spectrum(self, real, ncomp, tspec):
        if not self._pipelined(ncomp):
            self.b.forward(real, ncomp, self.send)
            self._exchange(ncomp)
            self.b.forward_finish(self.recv, ncomp, tspec)
            return
        # component c's exchange runs while component c + 1's 2D transform and
        # component c - 1's 1D transform do
        E, R, T = 2 * self.b.exch, self.b.real, 2 * self.b.tspec
        works = []
        for c in range(ncomp):
            self.b.forward(real[c * R:(c + 1) * R], 1, self.send[c * E:(c + 1) * E])
            works.append(self._a2a(self.recv[c * E:(c + 1) * E], self.send[c * E:(c + 1) * E]))
        for c in range(ncomp):
            works[c].wait()
            self.b.forward_finish(self.recv[c * E:(c + 1) * E], 1, tspec[c * T:(c + 1) * T])

    def _to_real(self, tspec, ncomp, real):
        if not self._pipelined(ncomp):
            self.b.inverse(tspec, ncomp, self.send)
            self._exchange(ncomp)
            self.b.inverse_finish(self.recv, ncomp, real)
            return
        E, R, T = 2 * self.b.exch, self.b.real, 2 * self.b.tspec
        works = []
        for c in range(ncomp):
            self.b.inverse(tspec[c * T:(c + 1) * T], 1, self.send[c * E:(c + 1) * E])
            works.append(self._a2a(self.recv[c * E:(c + 1) * E], self.send[c * E:(c + 1) * E]))
        for c in range(ncomp):
            works[c].wait()
            self.b.inverse_finish(self.recv[c * E:(c + 1) * E], 1, real[c * R:(c + 1) * R])

    def begin(self):
        """Bind the state and build the spectral copies of the initial state
        (stokes.py:363-370; Q^(0) = 0 is the gauge)."""
        cfg, st, be = self.cfg, self.state, self.b
        params = _params(cfg, self.pen, cfg.max_iter)
        be.begin(params, self.solid, st["u"], st["u_tilde"], st["q"], st["a"], st["lam"], self.hist)
        self._to_spectrum(st["q"], 1, self.TU)
        self._to_spectrum(st["u"], 3, self.TR)
        be.setup(self.TU, self.TR, self.Q, self.D)
        be.form_r(self.R, gated=False)
        self._to_spectrum(self.R, 3, self.TR)
        self.it = 0
        return self

    def iterate(self, n_iter: int, poll: bool = True) -> dict:
        """Up to ``n_iter`` more ADMM iterations (stokes.py:375-417); with
        ``poll`` the device control block is read every ``poll_every``
        iterations and the loop stops once it is done (identically on all ranks)."""
        be = self.b
        info = {"done": False}
        for _ in range(int(n_iter)):
            be.spectral(self.TR, self.Q, self.D, self.TU)
            self._to_real(self.TU, 3, self.unew)
            be.local(self.unew, self.totals)
            if self.world > 1:
                self.dist.all_reduce(self.totals, group=self.group)
            be.finalize(self.totals)
            be.form_r(self.R, gated=True)
            self.it += 1
            if poll and (self.it % self.poll == 0 or self.it == self.cfg.max_iter):
                info = be.read()
                if info["done"]:
                    return info
            self._to_spectrum(self.R, 3, self.TR)
        return info

    def end(self) -> ConvergenceReport:
        """q = Re ifft(Q^) into the state; the report (identical on all ranks)."""
        cfg, st, be = self.cfg, self.state, self.b
        info = be.read()
        n = float(np.prod(self.dims))
        be.scale(self.Q, self.TU, be.tspec, 1.0 / n)
        self._to_real(self.TU, 1, st["q"])
        its = info["iterations"]
        hist = self.hist[: its * len(REPORT_COLUMNS)].reshape(its, len(REPORT_COLUMNS))
        hist = hist.cpu().numpy() if hasattr(hist, "cpu") else np.asarray(hist)
        return ConvergenceReport(REPORT_COLUMNS, hist, converged=info["converged"], iterations=its,
                                 meta={"symbol_mode": cfg.symbol_mode, "eps_abs": cfg.eps_abs,
                                       "eps_rel": cfg.eps_rel, "nu": cfg.nu,
                                       "pressure_gradient": tuple(float(x) for x in cfg.pressure_gradient),
                                       "final_penalties": info["final_penalties"], "ranks": self.world,
                                       "pipeline": "slab"})

    def solve(self) -> ConvergenceReport:
        self.begin()
        self.iterate(self.cfg.max_iter, poll=True)
        return self.end()


class FusedSlabStokes(SlabStokes):
    """The same ADMM loop on the fused passes (csrc/pf_fused.cu): per iteration PK
    on this rank's y-slab of Y, an all-to-all of Y to the x-slab, the axis-1
    inverse + rows + local step (MI, RS), the 9-double all-reduce and finalize,
    the axis-1 forward (MF), and the all-to-all back.  Y is exchanged in the
    exchange-native layouts of ``pf_slab_fused_*`` (contiguous equal splits:
    one all_to_all per component plus one for the Nyquist columns, overlapped
    with the per-component passes), so there is no packing pass; at P = 1 both
    layouts coincide and nothing moves.  Only the Y buffers and the passes'
    own state stay resident: a cold start needs no transform (zero spectra),
    and the cuFFT-slab transforms of a warm start / the teardown exist only
    while they run — so a 1024^3 cell fits on two ranks."""

    def __init__(self, backend, dims, cfg, penalties, solid_local, state, group=None, poll_every: int = 8,
                 comm=None, overlap: bool = True, exchange: str = "a2a"):
        """``exchange``: "a2a" — all_to_all of the Y buffers between the passes
        (per component and overlapped when ``overlap``); "p2p" — the transpose
        fused into the passes: the Y buffers are P2P-mapped on every rank
        (``comm.p2p_alloc`` / ``p2p_ptrs``; torch symmetric memory on a GPU box,
        see ``SymmetricMemoryExchange``), PK and MF store their output straight
        into the owning ranks' buffers over NVLink, and a cross-rank barrier
        (``comm.p2p_barrier``) replaces each exchange.  "p2p" is EXPERIMENTAL: it is
        validated through the one-GPU loopback only; the two-GPU check
        (tests/test_gpu_slab_multi.py, tools/slab_multi_check.py) has not yet run on
        real NVLink peers."""
        super().__init__(backend, dims, cfg, penalties, solid_local, state, group, poll_every, comm, overlap)
        be = backend
        ym, yn = be.fused_sizes()
        if ym == 0:
            raise ValueError("fused slab pipeline unsupported for this grid / rank count")
        if exchange not in ("a2a", "p2p"):
            raise ValueError("exchange must be 'a2a' or 'p2p'")
        self.ym, self.yn = ym, yn
        self.p2p = exchange == "p2p" and self.world > 1
        if self.p2p:
            alloc = lambda k: self.dist.p2p_alloc(2 * k, backend.dev)  # noqa: E731
            self.Yy, self.Yyn, self.Yx, self.Yxn = alloc(ym), alloc(yn), alloc(ym), alloc(yn)
        else:
            self.Yy, self.Yyn = be.alloc_complex(ym), be.alloc_complex(yn)
            if self.world > 1:
                self.Yx, self.Yxn = be.alloc_complex(ym), be.alloc_complex(yn)
            else:
                self.Yx, self.Yxn = self.Yy, self.Yyn
        be.fused_bind(self.Yy, self.Yyn, self.Yx, self.Yxn)
        if self.p2p:
            ptrs = [self.dist.p2p_ptrs(t) for t in (self.Yy, self.Yyn, self.Yx, self.Yxn)]
            be.fused_set_peers(*ptrs)
        self._pending = []  # MF-side exchanges still in flight (overlapped mode)

    def _swap(self, src, srcn, dst, dstn):
        if self.world == 1:
            return
        per = 2 * self.ym // 3  # one component's main array (doubles)
        for c in range(3):
            self.dist.all_to_all_single(dst[c * per:(c + 1) * per], src[c * per:(c + 1) * per], group=self.group)
        self.dist.all_to_all_single(dstn, srcn, group=self.group)

    _eager_buffers = False  # the transform buffers exist only during setup / teardown

    def begin(self):
        cfg, st, be = self.cfg, self.state, self.b
        params = _params(cfg, self.pen, cfg.max_iter)
        be.begin(params, self.solid, st["u"], st["u_tilde"], st["q"], st["a"], st["lam"], self.hist)
        t = torch()
        nz = t.stack([t.count_nonzero(v) for v in st.values()]).sum().to(t.float64).reshape(1)
        if self.world > 1:  # every rank must take the same setup path (the transforms exchange)
            self.dist.all_reduce(nz, group=self.group)
        if float(nz.item()) == 0.0:
            be.fused_setup_zero()  # cold start: zero spectra and Y, no transform or scratch
        else:
            self._alloc_buffers(3)
            self._to_spectrum(st["q"], 1, self.TU)
            self._to_spectrum(st["u"], 3, self.TR)
            be.setup(self.TU, self.TR, self.Q, self.D)  # T-layout Q^ (gauged), D^
            be.fused_setup(self.Q, self.D, self.R)       # tile-major Q^, D^; x-slab Y of R; compact layout
            self._free_buffers()
            be.release_transforms()
            self._swap(self.Yx, self.Yxn, self.Yy, self.Yyn)
        if self.p2p:
            # the first PK stores into the peers' Yx: every rank's setup writes to
            # its own Y buffers (cold-start zeroing, the swap's reads) come first
            self.dist.p2p_barrier()
        self.it = 0
        return self

    def _drain(self):
        for w in self._pending:
            w.wait()
        self._pending = []

    def _comp(self, buf, c):
        per = 2 * self.ym // 3  # one component's main array (doubles)
        return buf[c * per:(c + 1) * per]

    def iterate(self, n_iter: int, poll: bool = True) -> dict:
        """Overlapped (P > 1, the default): after PK the Nyquist columns and the
        three components go out as four async all_to_alls and MI + RS of component
        c starts as soon as its data is in, under the transfer of c + 1; MF of
        component c is followed at once by its exchange back, under MF of c + 1;
        PK waits for all of them.  Same arithmetic as the blocking order."""
        be = self.b
        info = {"done": False}
        if self.p2p:
            return self._iterate_p2p(n_iter, poll)
        ov = self.overlap and self.world > 1
        for _ in range(int(n_iter)):
            self._drain()
            be.fused_pk()
            if ov:
                wn = self._a2a(self.Yxn, self.Yyn)
                ws = [self._a2a(self._comp(self.Yx, c), self._comp(self.Yy, c)) for c in range(3)]
                wn.wait()
                for c in range(3):
                    ws[c].wait()
                    be.fused_rs_part(c)
                be.fused_totals(self.totals)
            else:
                self._swap(self.Yy, self.Yyn, self.Yx, self.Yxn)
                be.fused_rs(self.totals)
            if self.world > 1:
                self.dist.all_reduce(self.totals, group=self.group)
            be.finalize(self.totals)
            if ov:
                for c in range(3):
                    be.fused_mf_part(c, c == 0)
                    self._pending.append(self._a2a(self._comp(self.Yy, c), self._comp(self.Yx, c)))
                self._pending.append(self._a2a(self.Yyn, self.Yxn))
            else:
                be.fused_mf()
            self.it += 1
            if poll and (self.it % self.poll == 0 or self.it == self.cfg.max_iter):
                info = be.read()
                if info["done"]:
                    return info  # (an exchange still in flight is drained by end(); Y is dead once done)
            if not ov:
                self._swap(self.Yx, self.Yxn, self.Yy, self.Yyn)
        return info

    def _iterate_p2p(self, n_iter: int, poll: bool) -> dict:
        """PK stores into the x-slab owners' Yx, MF into the y-slab owners' Yy;
        each barrier orders every rank's stores before the consuming pass (and,
        transitively, every rank's reads of a buffer before the next stores into it)."""
        be, d = self.b, self.dist
        info = {"done": False}
        for _ in range(int(n_iter)):
            be.fused_pk()
            d.p2p_barrier()
            be.fused_rs(self.totals)
            d.all_reduce(self.totals, group=self.group)
            be.finalize(self.totals)
            be.fused_mf()
            d.p2p_barrier()
            self.it += 1
            if poll and (self.it % self.poll == 0 or self.it == self.cfg.max_iter):
                info = be.read()
                if info["done"]:
                    return info
        return info

    def end(self) -> ConvergenceReport:
        self._drain()
        self._alloc_buffers(1, teardown=True)  # one component's transform buffers
        self.b.fused_end(self.Q)  # Q^ back to T layout; u~, a, lam materialised
        rep = super().end()
        self._free_buffers()
        self.b.release_transforms()
        rep.meta["pipeline"] = "slab-fused"
        rep.meta["exchange"] = "p2p" if self.p2p else ("a2a-overlapped" if self.overlap else "a2a")
        return rep


class SymmetricMemoryExchange:
    """torch.distributed with the peer-memory calls of the p2p exchange: Y buffers
    from torch symmetric memory (P2P-mapped into every rank over NVLink), their
    peer addresses from the rendezvous, and its device-side barrier (stream
    ordered, signal pads).  all_to_all_single / all_reduce go to the process group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        self.dist, self.symm, self.group = dist, symm_mem, group or dist.group.WORLD
        self.handles = {}

    def get_world_size(self, group=None):
        return self.dist.get_world_size(self.group)

    def get_rank(self, group=None):
        return self.dist.get_rank(self.group)

    def all_to_all_single(self, out, inp, group=None, async_op=False):
        return self.dist.all_to_all_single(out, inp, group=self.group, async_op=async_op)

    def all_reduce(self, t, group=None):
        return self.dist.all_reduce(t, group=self.group)

    def p2p_alloc(self, numel, device):
        t = torch()
        buf = self.symm.empty(numel, dtype=t.float64, device=device)
        self.handles[buf.data_ptr()] = self.symm.rendezvous(buf, self.group.group_name)
        return buf

    def p2p_ptrs(self, buf):
        return list(self.handles[buf.data_ptr()].buffer_ptrs)

    def p2p_barrier(self):
        next(iter(self.handles.values())).barrier(channel=0)


def slab_permeability(u_locals, solid_local, dims, symbol_mode: str = CENTRAL_MODE, group=None, device=None,
                      comm=None) -> np.ndarray:
    """K_ij = h^3 sum_pore sum_{c,m} d_m u^i_c d_m u^j_c (effective.py:43-72) of a
    slab-decomposed cell: ``u_locals`` = this rank's x-slabs (3, N0/P, N1, N2) of
    the three unit-flow solutions (e.g. from ``solve_stokes_slab``).  Each
    component goes through the distributed forward transform, its three spectral
    gradients back through the distributed inverse, the rank sums its masked Gram
    over its slab and the sums are all-reduced — no rank ever holds a whole field.
    Returns the same 3 x 3 tensor on every rank."""
    import torch.distributed as dist

    t = torch()
    if comm is not None:
        world, rank, d = comm.get_world_size(group), comm.get_rank(group), comm
    else:
        d = dist if dist.is_available() and dist.is_initialized() else None
        world = d.get_world_size(group) if d else 1
        rank = d.get_rank(group) if world > 1 else 0
    dims = tuple(int(x) for x in dims)
    if len(dims) != 3 or len(u_locals) != 3:
        raise ValueError("slab permeability needs three 3D unit-flow solutions")
    lo, hi = slab_range(dims[0], world, rank)
    be = DeviceSlabBackend(dims, world, rank, symbol_mode, device)
    be.bind()
    dev = be.dev
    L = (hi - lo) * dims[1] * dims[2]
    us = [t.as_tensor(np.asarray(u) if not hasattr(u, "data_ptr") else u).to(dev, t.float64).reshape(-1)
          for u in u_locals]
    for u in us:
        if u.numel() != 3 * L:
            raise ValueError("u_locals must be this rank's x-slab of each (3, N0, N1, N2) solution")
    solid = t.as_tensor(np.array(solid_local, dtype=np.uint8, copy=True)).reshape(-1).to(dev)
    tr = _SlabTransforms(be, world, d, group)
    spec = be.alloc_complex(be.tspec)
    grad = be.alloc_complex(be.tspec)
    G = be.alloc_real(9 * L)
    sums = np.zeros(6)
    for c in range(3):
        for i in range(3):
            tr.to_spectrum(us[i][c * L:(c + 1) * L], 1, spec)
            for m in range(3):
                be.grad(spec, m, grad)
                tr.to_real(grad, 1, G[(3 * i + m) * L:(3 * i + m + 1) * L])
        sums += be.gram(solid, G)
    tot = t.as_tensor(sums, dtype=t.float64, device=dev)
    if world > 1:
        d.all_reduce(tot, group=group)
    s6 = tot.cpu().numpy()
    be.close()
    cell = 1.0 / float(np.prod(dims))
    K = np.empty((3, 3))
    k = 0
    for i in range(3):
        for j in range(i, 3):
            K[i, j] = K[j, i] = s6[k] * cell
            k += 1
    return K


class _SlabTransforms:
    """Distributed 3D transforms of single components on a slab backend (forward:
    x-slab real -> T-layout spectrum; inverse: back), blocking exchanges."""

    def __init__(self, backend, world, dist, group):
        self.b, self.world, self.dist, self.group = backend, world, dist, group
        self.send = backend.alloc_complex(backend.exch)
        self.recv = backend.alloc_complex(backend.exch) if world > 1 else self.send

    def _exchange(self):
        if self.world > 1:
            self.dist.all_to_all_single(self.recv, self.send, group=self.group)

    def to_spectrum(self, real, ncomp, tspec):
        self.b.forward(real, ncomp, self.send)
        self._exchange()
        self.b.forward_finish(self.recv, ncomp, tspec)

    def to_real(self, tspec, ncomp, real):
        self.b.inverse(tspec, ncomp, self.send)
        self._exchange()
        self.b.inverse_finish(self.recv, ncomp, real)


def solve_stokes_slab(solid_local, dims, cfg: StokesConfig | None = None, penalties: PenaltyParams | None = None,
                      init_local: dict | None = None, group=None, device=None, comm=None, fused: bool | None = None,
                      overlap: bool = True, exchange: str = "a2a"):
    """Device slab solve on this rank: ``solid_local`` is the rank's x-slab of the
    indicator (uint8, (N0/P, N1, N2)); returns (local state dict of CUDA tensors,
    ConvergenceReport — identical on every rank)."""
    import torch.distributed as dist

    t = torch()
    cfg = cfg or StokesConfig(pressure_gradient=(1.0, 0.0, 0.0))
    if len(cfg.pressure_gradient) != 3 or len(dims) != 3:
        raise ValueError("slab decomposition is 3D")
    if comm is not None:
        world, rank = comm.get_world_size(group), comm.get_rank(group)
    else:
        world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
        rank = dist.get_rank(group) if world > 1 else 0
    lo, hi = slab_range(int(dims[0]), world, rank)
    if tuple(np.shape(solid_local)) != (hi - lo, int(dims[1]), int(dims[2])):
        raise ValueError("solid_local must be this rank's x-slab")
    be = DeviceSlabBackend(dims, world, rank, cfg.symbol_mode, device)
    be.bind()
    dev = be.dev
    L = (hi - lo) * int(dims[1]) * int(dims[2])
    if init_local is None:
        st = {k: t.zeros(3 * L, dtype=t.float64, device=dev) for k in ("u", "u_tilde", "a", "lam")}
        st["q"] = t.zeros(L, dtype=t.float64, device=dev)
    else:
        st = {k: t.as_tensor(np.asarray(init_local[k], dtype=np.float64)).reshape(-1).to(dev).clone()
              for k in ("u", "u_tilde", "q", "a", "lam")}
    solid = t.as_tensor(np.array(solid_local, dtype=np.uint8, copy=True)).reshape(-1).to(dev)
    if fused is None:
        fused = be.fused_sizes()[0] > 0
    cls = FusedSlabStokes if fused else SlabStokes
    kw = {"exchange": exchange} if fused else {}
    if fused and exchange == "p2p" and comm is None and world > 1:
        comm = SymmetricMemoryExchange(group)
    solver = cls(be, dims, cfg, penalties, solid, st, group, comm=comm, overlap=overlap, **kw)
    rep = solver.solve()
    t.cuda.synchronize(dev)
    shp3, shp1 = (3, hi - lo, int(dims[1]), int(dims[2])), (hi - lo, int(dims[1]), int(dims[2]))
    out = {k: (v.reshape(shp1) if k == "q" else v.reshape(shp3)) for k, v in st.items()}
    be.close()
    return out, rep

