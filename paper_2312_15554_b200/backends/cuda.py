"""The ``cuda`` kernel module: the five functions of reference
``backends/pure.py:26-115`` with identical signatures, computed by the
``pf_k_*`` entry points of libporeflow_b200.so.

Host (numpy) arrays in, fresh host arrays out; CUDA tensors in, CUDA tensors
out (no host round trip).  ``num_threads`` is accepted and ignored.
"""

from __future__ import annotations

import numpy as np

from .. import _native as N
from ..device import require_cuda, to_device, torch

NAME = "cuda"


def _dev(x, device, dtype):
    return to_device(x, device, dtype)


def _is_tensor(x):
    t = torch()
    return isinstance(x, t.Tensor)


def _out(x, host):
    return x.cpu().numpy() if host else x


def _stream(device):
    import ctypes

    return ctypes.c_void_p(torch().cuda.current_stream(device).cuda_stream)


def stokes_velocity_update(q_hat, a_hat, ut_hat, kappas, lap, kappa_sq, nu, beta, b, g_p, num_threads=1):
    """pure.py:26-56 (rank-one Green's operator per mode, full spectrum)."""
    host = not _is_tensor(q_hat)
    dev = require_cuda(None if host else q_hat.device)
    t = torch()
    c128 = t.complex128
    q = _dev(q_hat, dev, c128)
    a = _dev(a_hat, dev, c128)
    ut = _dev(ut_hat, dev, c128)
    ks = [_dev(np.asarray(k, dtype=np.float64) if not _is_tensor(k) else k, dev, t.float64) for k in kappas]
    L = _dev(lap, dev, t.float64)
    K2 = _dev(kappa_sq, dev, t.float64)
    out = t.empty_like(a)
    dims = tuple(q.shape)
    gp = N.dbl_array(np.asarray(g_p, dtype=float).ravel(), max(3, len(dims)))
    N.check(N.load().pf_k_stokes_velocity_update(
        len(dims), N.i64_array(dims), q.data_ptr(), a.data_ptr(), ut.data_ptr(),
        N.ptr_array([k.data_ptr() for k in ks]), L.data_ptr(), K2.data_ptr(), float(nu), float(beta), float(b),
        gp, out.data_ptr(), _stream(dev)))
    return _out(out, host)


def aux_velocity_update(u, a, lam, solid, alpha, b, num_threads=1):
    """pure.py:59-61."""
    host = not _is_tensor(u)
    dev = require_cuda(None if host else u.device)
    t = torch()
    f = t.float64
    U, A, L, S = (_dev(x, dev, f) for x in (u, a, lam, solid))
    out = t.empty_like(U)
    dims = tuple(S.shape)
    N.check(N.load().pf_k_aux_velocity_update(len(dims), N.i64_array(dims), U.data_ptr(), A.data_ptr(),
                                              L.data_ptr(), S.data_ptr(), float(alpha), float(b), out.data_ptr(),
                                              _stream(dev)))
    return _out(out, host)


def multiplier_update(a, lam, u, u_tilde, solid, alpha, b, num_threads=1):
    """pure.py:64-68."""
    host = not _is_tensor(a)
    dev = require_cuda(None if host else a.device)
    t = torch()
    f = t.float64
    A, L, U, UT, S = (_dev(x, dev, f) for x in (a, lam, u, u_tilde, solid))
    an, ln = t.empty_like(A), t.empty_like(L)
    dims = tuple(S.shape)
    N.check(N.load().pf_k_multiplier_update(len(dims), N.i64_array(dims), A.data_ptr(), L.data_ptr(), U.data_ptr(),
                                            UT.data_ptr(), S.data_ptr(), float(alpha), float(b), an.data_ptr(),
                                            ln.data_ptr(), _stream(dev)))
    return _out(an, host), _out(ln, host)


def transport_polarization(grad_chi, diffusivity, advection, forcing, a0, b0_vec, g_chi, num_threads=1):
    """pure.py:71-87."""
    host = not _is_tensor(grad_chi)
    dev = require_cuda(None if host else grad_chi.device)
    t = torch()
    f = t.float64
    G, Df, Ad, F = (_dev(x, dev, f) for x in (grad_chi, diffusivity, advection, forcing))
    w, s = t.empty_like(G), t.empty_like(F)
    dims = tuple(F.shape)
    b0 = N.dbl_array(np.asarray(b0_vec, dtype=float).ravel(), 3)
    gc = N.dbl_array(np.asarray(g_chi, dtype=float).ravel(), 3)
    N.check(N.load().pf_k_transport_polarization(len(dims), N.i64_array(dims), G.data_ptr(), Df.data_ptr(),
                                                 Ad.data_ptr(), F.data_ptr(), float(a0), b0, gc, w.data_ptr(),
                                                 s.data_ptr(), _stream(dev)))
    return _out(w, host), _out(s, host)


def transport_mode_update(w_hat, s_hat, kappas, lap, a0, b0_vec, num_threads=1):
    """pure.py:90-115."""
    host = not _is_tensor(s_hat)
    dev = require_cuda(None if host else s_hat.device)
    t = torch()
    c128 = t.complex128
    W, S = _dev(w_hat, dev, c128), _dev(s_hat, dev, c128)
    ks = [_dev(np.asarray(k, dtype=np.float64) if not _is_tensor(k) else k, dev, t.float64) for k in kappas]
    L = _dev(lap, dev, t.float64)
    chi, grad = t.empty_like(S), t.empty_like(W)
    dims = tuple(S.shape)
    b0 = N.dbl_array(np.asarray(b0_vec, dtype=float).ravel(), 3)
    N.check(N.load().pf_k_transport_mode_update(len(dims), N.i64_array(dims), W.data_ptr(), S.data_ptr(),
                                                N.ptr_array([k.data_ptr() for k in ks]), L.data_ptr(), float(a0),
                                                b0, chi.data_ptr(), grad.data_ptr(), _stream(dev)))
    return _out(chi, host), _out(grad, host)
