"""Device mechanics behind the reference's transform utilities and step helpers
(``spectral.fft/ifft/grad/div/apply_laplacian/gradient_field``,
``stokes.step1/2/3``, ``residuals_and_tolerances``, ``transport.residual_rhs`` and
``update_concentration``): CUDA tensors in, CUDA tensors out, every operation a
``pf_k_*`` entry point of libporeflow_b200.so (``csrc/pf_ops.cu``).

The public wrappers accept numpy arrays (copied in, results copied back as
fresh arrays, the reference's ownership rule: inputs are never mutated) or CUDA
tensors (kept on the device).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .device import require_cuda, to_device, torch


def is_tensor(x) -> bool:
    return isinstance(x, torch().Tensor)


def device_of(*xs):
    for x in xs:
        if is_tensor(x):
            return require_cuda(x.device)
    return require_cuda(None)


def stream(dev):
    return ctypes.c_void_p(torch().cuda.current_stream(dev).cuda_stream)


def real(x, dev):
    return to_device(x, dev, torch().float64)


def cplx(x, dev):
    t = torch()
    if is_tensor(x):
        return x.to(device=dev, dtype=t.complex128).contiguous()
    return to_device(np.asarray(x, dtype=np.complex128), dev, t.complex128)


def out_like(x_dev, host: bool):
    return x_dev.cpu().numpy() if host else x_dev


def kappa_tables(symbols, dev):
    return [real(np.asarray(k, dtype=np.float64) if not is_tensor(k) else k, dev) for k in symbols.kappa]


def _split(shape, ndim):
    grid = tuple(int(n) for n in shape[len(shape) - ndim:])
    batch = int(np.prod(shape[: len(shape) - ndim], dtype=np.int64)) if len(shape) > ndim else 1
    return grid, batch


def fftn_t(x, ndim: int):
    """Full complex forward transform over the trailing ``ndim`` axes."""
    t = torch()
    dev = require_cuda(x.device)
    dims, batch = _split(tuple(x.shape), ndim)
    is_c = x.is_complex()
    src = x.contiguous() if is_c else x.to(t.float64).contiguous()
    out = t.empty(tuple(x.shape), dtype=t.complex128, device=dev)
    if batch * int(np.prod(dims)) == 0:
        return out
    N.check(N.load().pf_k_fftn(ndim, N.i64_array(dims), batch, src.data_ptr(), int(is_c), out.data_ptr(), 0,
                               stream(dev)))
    return out


def ifftn_real_t(z, ndim: int):
    """Re ifftn over the trailing ``ndim`` axes (1/n folded in)."""
    t = torch()
    dev = require_cuda(z.device)
    dims, batch = _split(tuple(z.shape), ndim)
    src = z.to(t.complex128).contiguous()
    work = t.empty_like(src)
    out = t.empty(tuple(z.shape), dtype=t.float64, device=dev)
    if out.numel() == 0:
        return out
    N.check(N.load().pf_k_ifftn_real(ndim, N.i64_array(dims), batch, src.data_ptr(), work.data_ptr(),
                                     out.data_ptr(), stream(dev)))
    return out


def grad_t(chi_hat, kaps, ndim: int):
    t = torch()
    dev = require_cuda(chi_hat.device)
    dims, batch = _split(tuple(chi_hat.shape), ndim)
    src = chi_hat.to(t.complex128).contiguous()
    out = t.empty((ndim,) + tuple(chi_hat.shape), dtype=t.complex128, device=dev)
    N.check(N.load().pf_k_spectral_grad(ndim, N.i64_array(dims), batch, N.ptr_array([k.data_ptr() for k in kaps]),
                                        src.data_ptr(), out.data_ptr(), stream(dev)))
    return out


def div_t(v_hat, kaps, ndim: int, base=None):
    t = torch()
    dev = require_cuda(v_hat.device)
    if v_hat.dim() != ndim + 1 or v_hat.shape[0] != ndim:
        raise ValueError(f"div expects a ({ndim}, *dims) spectral vector field, got shape {tuple(v_hat.shape)}")
    dims = tuple(int(n) for n in v_hat.shape[1:])
    src = v_hat.to(t.complex128).contiguous()
    b = base.to(t.complex128).contiguous() if base is not None else None
    out = t.empty(dims, dtype=t.complex128, device=dev)
    N.check(N.load().pf_k_spectral_div(ndim, N.i64_array(dims), N.ptr_array([k.data_ptr() for k in kaps]),
                                       src.data_ptr(), b.data_ptr() if b is not None else None, out.data_ptr(),
                                       stream(dev)))
    return out


def scale_modes_t(factor, z, sign: float):
    """(sign*factor) * z, factor broadcast over z's leading axes."""
    t = torch()
    dev = require_cuda(z.device)
    f = factor.to(device=dev, dtype=t.float64).contiguous()
    src = z.to(t.complex128).contiguous()
    nm = f.numel()
    if src.numel() % nm or tuple(src.shape[src.dim() - f.dim():]) != tuple(f.shape):
        raise ValueError("symbol shape does not match the trailing axes of the spectral field")
    out = t.empty_like(src)
    N.check(N.load().pf_k_scale_modes(nm, src.numel() // nm, f.data_ptr(), float(sign), src.data_ptr(),
                                      out.data_ptr(), stream(dev)))
    return out


def _scratch(dev):
    t = torch()
    return t.empty(int(N.load().pf_k_scratch_doubles()), dtype=t.float64, device=dev)


def q_update_t(q, div_u, beta: float):
    t = torch()
    dev = require_cuda(q.device)
    qq, dd = q.to(t.float64).contiguous(), div_u.to(t.float64).contiguous()
    out = t.empty_like(qq)
    N.check(N.load().pf_k_q_update(qq.numel(), qq.data_ptr(), dd.data_ptr(), float(beta), out.data_ptr(),
                                   _scratch(dev).data_ptr(), stream(dev)))
    return out


def norm_t(x, y=None, w=None) -> float:
    """||w*(x - y)||_2 with w a scalar field broadcast over x's leading axis."""
    t = torch()
    dev = require_cuda(x.device)
    xx = x.to(t.float64).contiguous()
    yy = y.to(t.float64).contiguous() if y is not None else None
    ww = w.to(t.float64).contiguous() if w is not None else None
    if yy is not None and yy.shape != xx.shape:
        raise ValueError("norm operands differ in shape")
    res = ctypes.c_double(0.0)
    N.check(N.load().pf_k_norm(xx.numel(), xx.data_ptr(), yy.data_ptr() if yy is not None else None,
                               ww.data_ptr() if ww is not None else None, ww.numel() if ww is not None else 1,
                               _scratch(dev).data_ptr(), ctypes.byref(res), stream(dev)))
    return float(res.value)
