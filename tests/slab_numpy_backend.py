"""TEST DOUBLE: numpy implementation of the per-rank slab operations
(the pf_slab_* device work), used to exercise the product's slab driver
(paper_2312_15554_b200/slab.py) over gloo on CPU.  Mirrors the device
semantics: unnormalised transforms, 1/n folded into U^, half-spectrum
Parseval sums, the finalize decisions of stokes.py:247-310."""

import math

import numpy as np
import torch

from oracle import poreflow_oracle as O


class NumpySlabBackend:
    def __init__(self, dims, world, rank, mode="central"):
        self.N0, self.N1, self.N2 = dims
        self.P, self.rank = world, rank
        self.L0, self.L1, self.H2 = self.N0 // world, self.N1 // world, self.N2 // 2 + 1
        self.exch = self.P * self.L0 * self.L1 * self.H2
        self.tspec = self.N0 * self.L1 * self.H2
        self.real = self.L0 * self.N1 * self.N2
        kap, _, _ = O.symbols(dims, mode)
        lap1 = []
        for ax, n in enumerate(dims):
            h = 1.0 / n
            k = 2.0 * np.pi * np.fft.fftfreq(n, d=1.0 / n)
            lap1.append(k ** 2 if mode == "exact" else 4.0 * np.sin(0.5 * h * k) ** 2 / h ** 2)
        off = rank * self.L1
        self.k0 = kap[0][:, None, None]
        self.k1 = kap[1][off:off + self.L1][None, :, None]
        self.k2 = kap[2][: self.H2][None, None, :]
        self.lap = (lap1[0][:, None, None] + lap1[1][off:off + self.L1][None, :, None]) + lap1[2][: self.H2][None, None, :]
        self.ksq = (self.k0 ** 2 + self.k1 ** 2) + self.k2 ** 2
        w = np.full(self.H2, 2.0)
        w[0] = 1.0
        if self.N2 % 2 == 0:
            w[-1] = 1.0
        self.w = w[None, None, :]
        self.n = float(self.N0 * self.N1 * self.N2)

    # buffers
    def alloc_complex(self, count):
        return torch.zeros(2 * count, dtype=torch.float64)

    def alloc_real(self, count):
        return torch.zeros(count, dtype=torch.float64)

    @staticmethod
    def c(x, shape):
        return x.numpy().view(np.complex128)[: int(np.prod(shape))].reshape(shape)

    @staticmethod
    def r(x, shape):
        return x.numpy()[: int(np.prod(shape))].reshape(shape)

    # transforms + exchange packing
    def forward(self, real, ncomp, send):
        A = np.fft.rfftn(self.r(real, (ncomp, self.L0, self.N1, self.N2)), axes=(2, 3))
        S = self.c(send, (self.P, ncomp, self.L0, self.L1, self.H2))
        for s in range(self.P):
            S[s] = A[:, :, s * self.L1:(s + 1) * self.L1, :]

    def forward_finish(self, recv, ncomp, tspec):
        Rv = self.c(recv, (self.P, ncomp, self.L0, self.L1, self.H2))
        T = self.c(tspec, (ncomp, self.N0, self.L1, self.H2))
        for s in range(self.P):
            T[:, s * self.L0:(s + 1) * self.L0] = Rv[s]
        T[...] = np.fft.fft(T, axis=1)

    def inverse(self, tspec, ncomp, send):
        T = self.c(tspec, (ncomp, self.N0, self.L1, self.H2))
        T[...] = np.fft.ifft(T, axis=1, norm="forward")
        S = self.c(send, (self.P, ncomp, self.L0, self.L1, self.H2))
        for s in range(self.P):
            S[s] = T[:, s * self.L0:(s + 1) * self.L0]

    def inverse_finish(self, recv, ncomp, real):
        Rv = self.c(recv, (self.P, ncomp, self.L0, self.L1, self.H2))
        A = np.empty((ncomp, self.L0, self.N1, self.H2), complex)
        for s in range(self.P):
            A[:, :, s * self.L1:(s + 1) * self.L1, :] = Rv[s]
        self.r(real, (ncomp, self.L0, self.N1, self.N2))[...] = np.fft.irfftn(A, s=(self.N1, self.N2), axes=(2, 3),
                                                                               norm="forward")

    # solver steps
    def begin(self, params, solid, u, ut, q, a, lam, hist):
        self.p = params
        self.solid = solid.numpy().reshape(self.L0, self.N1, self.N2).astype(float)
        self.st = dict(u=u, ut=ut, q=q, a=a, lam=lam)
        self.hist = hist
        self.ctrl = dict(alpha=params.alpha, beta=params.beta, b=params.b, iter=0, done=False, converged=False)
        self.part1 = np.zeros(3)

    def setup(self, Tq, Tu, Q, D):
        Qv = self.c(Q, (self.N0, self.L1, self.H2))
        Qv[...] = self.c(Tq, (self.N0, self.L1, self.H2))
        if self.rank == 0:
            Qv[0, 0, 0] = 0.0
        Uv = self.c(Tu, (3, self.N0, self.L1, self.H2))
        self.c(D, (self.N0, self.L1, self.H2))[...] = 1j * self.k0 * Uv[0] + 1j * self.k1 * Uv[1] + 1j * self.k2 * Uv[2]

    def spectral(self, R, Q, D, U):
        if self.ctrl["done"]:
            return
        beta, b = self.ctrl["beta"], self.ctrl["b"]
        Rv = self.c(R, (3, self.N0, self.L1, self.H2))
        Qv = self.c(Q, (self.N0, self.L1, self.H2))
        Dv = self.c(D, (self.N0, self.L1, self.H2))
        ks = (self.k0, self.k1, self.k2)
        r = [-1j * ks[c] * Qv + Rv[c] for c in range(3)]
        if self.rank == 0:
            for c in range(3):
                r[c][0, 0, 0] += self.n * self.p.pressure_gradient[c]
        A = self.p.nu * self.lap + b
        kr = ks[0] * r[0] + ks[1] * r[1] + ks[2] * r[2]
        corr = beta / (A + beta * self.ksq) * kr
        u = [(r[c] - ks[c] * corr) / A for c in range(3)]
        dv = 1j * ks[0] * u[0] + 1j * ks[1] * u[1] + 1j * ks[2] * u[2]
        qn = Qv - beta * dv
        if self.rank == 0:
            qn[0, 0, 0] = 0.0
        self.part1 = np.array([(self.w * abs(dv) ** 2).sum(), (self.w * abs(dv - Dv) ** 2).sum(),
                               (self.w * abs(qn) ** 2).sum()])
        Qv[...] = qn
        Dv[...] = dv
        Uv = self.c(U, (3, self.N0, self.L1, self.H2))
        for c in range(3):
            Uv[c] = u[c] / self.n

    def local(self, unew, totals):
        tv = totals.numpy()
        if self.ctrl["done"]:
            return
        sh = (3, self.L0, self.N1, self.N2)
        u1 = self.r(unew, sh)
        u, ut, a, lam = (self.r(self.st[k], sh) for k in ("u", "ut", "a", "lam"))
        H = self.solid
        alpha, b = self.ctrl["alpha"], self.ctrl["b"]
        t1 = O.aux_velocity_update(u1, a, lam, H, alpha, b)
        a1, l1 = O.multiplier_update(a, lam, u1, t1, H, alpha, b)
        sums = [((H * t1) ** 2).sum(), ((H * (t1 - ut)) ** 2).sum(), (l1 ** 2).sum(), ((u1 - t1) ** 2).sum(),
                ((u1 - u) ** 2).sum(), (a1 ** 2).sum()]
        u[...], ut[...], a[...], lam[...] = u1, t1, a1, l1
        tv[:6] = sums
        tv[6:] = self.part1

    def finalize(self, totals):
        c = self.ctrl
        if c["done"]:
            return
        S = totals.numpy()
        al, be, b = c["alpha"], c["beta"], c["b"]
        er = self.p.eps_rel
        tv = math.sqrt(3 * self.n) * self.p.eps_abs
        ts = math.sqrt(self.n) * self.p.eps_abs
        rp1, rd1, ln = math.sqrt(S[0]), al * math.sqrt(S[1]), math.sqrt(S[2])
        rp2, rd2, qn = math.sqrt(S[6] / self.n), be * math.sqrt(S[7] / self.n), math.sqrt(S[8] / self.n)
        rp3, rd3, an = math.sqrt(S[3]), b * math.sqrt(S[4]), math.sqrt(S[5])
        pairs = ((rp1, tv + er * max(rp1, ln), rd1, tv + er * ln), (rp2, ts + er * max(rp2, qn), rd2, ts + er * qn),
                 (rp3, tv + er * max(rp3, an), rd3, tv + er * an))
        row = [x for pr in pairs for x in pr] + [al, be, b]
        it = c["iter"] + 1
        self.hist.numpy()[(it - 1) * 15: it * 15] = row
        c["iter"] = it
        if all(pr[0] <= pr[1] and pr[2] <= pr[3] for pr in pairs):
            c["done"] = c["converged"] = True
            return
        if self.p.adaptive:
            pen = dict(alpha=al, beta=be, b=b, growth=tuple(self.p.growth), ratio_threshold=tuple(self.p.ratio_threshold),
                       floor=tuple(self.p.floor))
            out = O.adapt(pen, pairs)
            c["alpha"], c["beta"], c["b"] = out["alpha"], out["beta"], out["b"]
        if it >= self.p.max_iter:
            c["done"] = True

    def form_r(self, R, gated):
        if gated and self.ctrl["done"]:
            return
        sh = (3, self.L0, self.N1, self.N2)
        self.r(R, sh)[...] = self.ctrl["b"] * self.r(self.st["ut"], sh) - self.r(self.st["a"], sh)

    def scale(self, src, dst, count, s):
        dst.numpy()[: 2 * count] = src.numpy()[: 2 * count] * s

    def read(self):
        c = self.ctrl
        return {"iterations": c["iter"], "converged": c["converged"], "done": c["done"],
                "final_penalties": (c["alpha"], c["beta"], c["b"])}
