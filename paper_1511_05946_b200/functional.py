"""Tensor-level entry points over the C ABI, plus the autograd Function.

Every op launches on ``torch.cuda.current_stream()`` of the input's device and
returns without synchronising.  Inputs must be CUDA fp32 tensors whose rows
are contiguous (stride(-1) == 1); anything else is made contiguous first.

Reference counterparts (under /root/reference/pkg/src/acdc):
  acdc_forward   AcdcLayer.forward   layers.py:141-146
  acdc_backward  AcdcLayer.backward  layers.py:148-156 (accumulating grads)
  dct / idct     transforms.py:137-156
"""

from __future__ import annotations

import contextlib
import ctypes
import os

import torch

from . import _lib

__all__ = [
    "acdc_forward",
    "acdc_backward",
    "acdc_backward_sgd",
    "acdc_step",
    "step_max_rows",
    "dct",
    "fft",
    "ifft",
    "idct",
    "AcdcFunction",
    "acdc",
    "afdf_forward",
    "afdf_backward",
    "AfdfFunction",
    "afdf",
    "prepare",
    "h2cache_supported",
    "new_h2cache",
    "cascade_supported",
    "cascade_forward",
    "cascade_backward",
    "HostPipeline",
    "relu_forward",
    "relu_backward",
    "gather_cols",
]


_NULLCTX = contextlib.nullcontext()


def _on(dev: torch.device):
    """Make ``dev`` current for the C call; no context switch (two cudaSetDevice
    calls) when it already is -- the common case, and a measurable share of a
    small call's host time."""
    return _NULLCTX if dev.index is None or dev.index == torch.cuda.current_device() else torch.cuda.device(dev)


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _rows2d(x: torch.Tensor, n: int, name: str = "x") -> torch.Tensor:
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if x.dim() != 2 or x.shape[1] != n:
        raise ValueError(f"{name} must have shape (batch, {n}), got {tuple(x.shape)}")
    if x.dtype != torch.float32:
        x = x.float()
    if x.stride(1) != 1 or (x.shape[0] > 1 and x.stride(0) < n):
        x = x.contiguous()
    elif n >= 1024 and x.numel() and (x.data_ptr() % 16 or (x.shape[0] > 1 and x.stride(0) % 4)):
        x = x.contiguous()  # the half-length-plan kernels (n >= 1024) move rows as 128-bit quads
    return x


def _vec(v: torch.Tensor, n: int, dev, name: str) -> torch.Tensor:
    if v.dim() != 1 or v.shape[0] != n:
        raise ValueError(f"{name} must have shape ({n},), got {tuple(v.shape)}")
    if v.device != dev or v.dtype != torch.float32 or not v.is_contiguous():
        v = v.to(device=dev, dtype=torch.float32).contiguous()
    return v


def _ld(x: torch.Tensor, n: int) -> int:
    return x.stride(0) if x.shape[0] > 1 else n


def _check_out(out: torch.Tensor, like: torch.Tensor, name: str = "out", host_ok: bool = False) -> torch.Tensor:
    """A caller-supplied output must match ``like``: shape, dtype, rows with
    unit stride and a row stride the kernels can use, and (unless it is a
    pinned host buffer the kernels store to directly) the input's device."""
    if not isinstance(out, torch.Tensor) or out.shape != like.shape or out.dtype != like.dtype:
        raise ValueError(f"{name} must be a {like.dtype} tensor of shape {tuple(like.shape)}")
    if out.dim() == 2 and out.shape[0] > 0 and (out.stride(1) != 1 or (out.shape[0] > 1 and out.stride(0) < out.shape[1])):
        raise ValueError(f"{name} rows must be contiguous with row stride >= {out.shape[1]}")
    if out.device != like.device and not (host_ok and out.device.type == "cpu" and out.is_pinned()):
        raise ValueError(f"{name} must be on {like.device}")
    return out


def _check_h2cache(h2cache: torch.Tensor, rows: int, n: int, dev) -> torch.Tensor:
    need = _lib.load().acdc_h2cache_bytes(rows, n)
    if need == 0:
        raise ValueError(f"the h2 cache needs 256 <= n <= 32768, got {n}")
    if (not isinstance(h2cache, torch.Tensor) or h2cache.device != dev or h2cache.dtype != torch.float32
            or not h2cache.is_contiguous() or h2cache.numel() * 4 < need):
        raise ValueError(f"h2cache must be a contiguous fp32 tensor on {dev} of at least {need} bytes "
                         f"(new_h2cache({rows}, {n}))")
    return h2cache


def prepare(n: int, device=None) -> None:
    """Build tables and launch configuration for size n (call before graph capture)."""
    with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
        _lib.check(_lib.load().acdc_prepare(int(n)))


def h2cache_supported(n: int) -> bool:
    """Sizes whose kernels can cache h2 = C2(a*x) between forward and backward
    (256 <= n <= 16384 on the row-pair kernels, up to 32768 on the half-length plan)."""
    return 256 <= n <= 32768 and (n & (n - 1)) == 0 and _lib.load().acdc_h2cache_bytes(2, n) > 0


def new_h2cache(rows: int, n: int, device) -> torch.Tensor:
    """Buffer for the h2 cache of ``rows`` rows (opaque, kernel-native layout)."""
    nbytes = _lib.load().acdc_h2cache_bytes(rows, n)
    if nbytes == 0:
        raise ValueError(f"the h2 cache needs 256 <= n <= 32768, got {n}")
    return torch.empty(nbytes // 4, dtype=torch.float32, device=device)


def acdc_forward(x: torch.Tensor, a: torch.Tensor, d: torch.Tensor, bias: torch.Tensor, out=None,
                 h2cache: torch.Tensor | None = None) -> torch.Tensor:
    """y = C3(d * C2(a * x) + bias) row-wise (layers.py:141-146).

    With ``h2cache`` (from :func:`new_h2cache`) the kernel also stores
    h2 = C2(a * x) for :func:`acdc_backward`, like the reference's cache
    (layers.py:145)."""
    n = a.shape[0]
    x = _rows2d(x, n)
    dev = x.device
    a, d, bias = (_vec(v, n, dev, nm) for v, nm in ((a, "a"), (d, "d"), (bias, "bias")))
    y = torch.empty_like(x, memory_format=torch.contiguous_format) if out is None else _check_out(out, x, host_ok=True)
    if h2cache is not None:
        _check_h2cache(h2cache, x.shape[0], n, dev)
    lib = _lib.load()
    with _on(dev):
        if h2cache is None:
            rc = lib.acdc_fwd_f32(_ptr(x), _ptr(y), _ptr(a), _ptr(d), _ptr(bias), x.shape[0], n, _ld(x, n), _ld(y, n),
                                  _stream(x))
        else:
            rc = lib.acdc_fwd_cache_f32(_ptr(x), _ptr(y), _ptr(a), _ptr(d), _ptr(bias), _ptr(h2cache), x.shape[0], n,
                                        _ld(x, n), _ld(y, n), _stream(x))
        _lib.check(rc)
    return y


def step_max_rows(n: int) -> int:
    """Largest batch :func:`acdc_step` runs as one fused launch at size n (0: none)."""
    return int(_lib.load().acdc_step_max_rows(int(n)))


def acdc_step(x: torch.Tensor, dy: torch.Tensor, a: torch.Tensor, d: torch.Tensor, bias: torch.Tensor,
              grad_a: torch.Tensor, grad_d: torch.Tensor, grad_bias: torch.Tensor, accumulate: bool = True,
              out_y=None, out_dx=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Forward and backward of one layer for an upstream gradient ``dy`` known
    before the forward (AcdcLayer.forward then .backward, layers.py:141-156):
    returns (y, dx) and updates the gradients like :func:`acdc_backward`.

    Up to :func:`step_max_rows` rows (small batches, 256 <= n <= 2048) this is
    ONE kernel launch (forward, backward and the gradient reduction in one
    CTA); larger batches run :func:`acdc_forward` + :func:`acdc_backward`."""
    n = a.shape[0]
    x = _rows2d(x, n)
    dy = _rows2d(dy, n, "grad_y")
    if dy.shape[0] != x.shape[0]:
        raise ValueError(f"grad_y has {dy.shape[0]} rows, input had {x.shape[0]}")
    rows = x.shape[0]
    if rows > step_max_rows(n):
        y = acdc_forward(x, a, d, bias, out=out_y)
        return y, acdc_backward(x, dy, a, d, grad_a, grad_d, grad_bias, accumulate=accumulate, out=out_dx)
    dev = x.device
    a, d, bias = (_vec(v, n, dev, nm) for v, nm in ((a, "a"), (d, "d"), (bias, "bias")))
    for g in (grad_a, grad_d, grad_bias):
        if g.device != dev or g.dtype != torch.float32 or not g.is_contiguous() or g.shape != (n,):
            raise ValueError("gradient buffers must be contiguous fp32 (n,) tensors on the input device")
    y = torch.empty_like(x, memory_format=torch.contiguous_format) if out_y is None else _check_out(out_y, x, "out_y")
    dx = torch.empty_like(x, memory_format=torch.contiguous_format) if out_dx is None else _check_out(out_dx, x, "out_dx")
    lib = _lib.load()
    with _on(dev):
        _lib.check(lib.acdc_step_f32(_ptr(x), _ptr(dy), _ptr(y), _ptr(dx), _ptr(a), _ptr(d), _ptr(bias), _ptr(grad_a),
                                     _ptr(grad_d), _ptr(grad_bias), 1 if accumulate else 0, rows, n, _ld(x, n),
                                     _ld(dy, n), _ld(y, n), _ld(dx, n), _stream(x)))
    return y, dx


def acdc_backward(
    x: torch.Tensor,
    dy: torch.Tensor,
    a: torch.Tensor,
    d: torch.Tensor,
    grad_a: torch.Tensor,
    grad_d: torch.Tensor,
    grad_bias: torch.Tensor,
    accumulate: bool = True,
    out=None,
    h2cache: torch.Tensor | None = None,
) -> torch.Tensor:
    """dx and (accumulated) parameter gradients of acdc_forward (layers.py:148-156).

    grad_a / grad_d / grad_bias are CUDA fp32 (n,) tensors updated in place:
    ``+=`` when ``accumulate`` (the reference contract), ``=`` otherwise.
    ``h2cache`` (filled by the matching forward) skips recomputing C2(a * x).
    """
    n = a.shape[0]
    x = _rows2d(x, n)
    dy = _rows2d(dy, n, "grad_y")
    if dy.shape[0] != x.shape[0]:
        raise ValueError(f"grad_y has {dy.shape[0]} rows, input had {x.shape[0]}")
    dev = x.device
    a, d = _vec(a, n, dev, "a"), _vec(d, n, dev, "d")
    for g in (grad_a, grad_d, grad_bias):
        if g.device != dev or g.dtype != torch.float32 or not g.is_contiguous() or g.shape != (n,):
            raise ValueError("gradient buffers must be contiguous fp32 (n,) tensors on the input device")
    dx = torch.empty_like(x, memory_format=torch.contiguous_format) if out is None else _check_out(out, x, host_ok=True)
    if h2cache is not None:
        _check_h2cache(h2cache, x.shape[0], n, dev)
    lib = _lib.load()
    with _on(dev):
        wsb = lib.acdc_bwd_workspace_bytes(x.shape[0], n)
        if wsb == 0:
            _lib.check(_lib.ACDC_E_CUDA)
        ws = torch.empty((wsb + 3) // 4, dtype=torch.float32, device=dev)
        common = (1 if accumulate else 0, _ptr(ws), wsb, x.shape[0], n, _ld(x, n), _ld(dy, n), _ld(dx, n), _stream(x))
        if h2cache is None:
            rc = lib.acdc_bwd_f32(_ptr(x), _ptr(dy), _ptr(dx), _ptr(a), _ptr(d), _ptr(grad_a), _ptr(grad_d),
                                  _ptr(grad_bias), *common)
        else:
            rc = lib.acdc_bwd_cached_f32(_ptr(x), _ptr(dy), _ptr(dx), _ptr(a), _ptr(d), _ptr(h2cache), _ptr(grad_a),
                                         _ptr(grad_d), _ptr(grad_bias), *common)
        _lib.check(rc)
    return dx


def acdc_backward_sgd(x, dy, params, velocities, lr, weight_decay, momentum, grads=None, accumulate=False, out=None,
                      h2cache=None, prev_perm=None, prev_relu=False, ws=None, h2_rowpair=False) -> torch.Tensor:
    """Backward of one ACDC layer fused with its momentum-SGD step (reference
    AcdcLayer.backward + Sgd.step, layers.py:148-156, training.py:58-98).

    ``params`` = (a, d, bias_d) and ``velocities`` are fp32 (n,) CUDA tensors
    updated in place; ``lr`` / ``weight_decay``: 3 floats (lr_t * lr_mult and
    the decay actually applied, per parameter).  ``grads`` (grad_a, grad_d,
    grad_bias) are added to the batch gradient when ``accumulate`` and zeroed.
    ``h2cache`` / ``prev_perm`` / ``prev_relu`` select the cached and fused-
    cascade block backward (``h2_rowpair``: the cache was written by the fused
    cascade forward).  Returns dx (computed with the pre-step a, d)."""
    a = params[0]
    n = a.shape[0]
    x = _rows2d(x, n)
    dy = _rows2d(dy, n, "grad_y")
    if dy.shape[0] != x.shape[0]:
        raise ValueError(f"grad_y has {dy.shape[0]} rows, input had {x.shape[0]}")
    dev = x.device
    for t in (*params, *velocities, *(grads or ())):
        if t.device != dev or t.dtype != torch.float32 or not t.is_contiguous() or t.shape != (n,):
            raise ValueError("parameter, velocity and gradient buffers must be contiguous fp32 (n,) tensors")
    if accumulate and grads is None:
        raise ValueError("accumulate=True needs the gradient buffers")
    dx = torch.empty_like(x, memory_format=torch.contiguous_format) if out is None else _check_out(out, x)
    if h2cache is not None:
        _check_h2cache(h2cache, x.shape[0], n, dev)
    st = _lib.SgdStep()
    for k in range(3):
        st.value[k] = params[k].data_ptr()
        st.velocity[k] = velocities[k].data_ptr()
        st.lr[k] = float(lr[k])
        st.weight_decay[k] = float(weight_decay[k])
    st.momentum = float(momentum)
    g = grads if grads is not None else (None, None, None)
    lib = _lib.load()
    with _on(dev):
        wsb = lib.acdc_bwd_workspace_bytes(max(x.shape[0], 1), n)
        if wsb == 0:
            _lib.check(_lib.ACDC_E_CUDA)
        if ws is None or ws.numel() * 4 < wsb:
            ws = torch.empty((wsb + 3) // 4, dtype=torch.float32, device=dev)
        _lib.check(lib.acdc_bwd_sgd_f32(
            _ptr(x), _ptr(dy), _ptr(dx), _ptr(h2cache), _ptr(prev_perm), (1 if prev_relu else 0) | (2 if h2_rowpair else 0),
            _ptr(g[0]),
            _ptr(g[1]), _ptr(g[2]), 1 if accumulate else 0, ctypes.byref(st), _ptr(ws), wsb, x.shape[0], n,
            _ld(x, n), _ld(dy, n), _ld(dx, n), _stream(x)))
    return dx


def _transform(fn_name: str, x: torch.Tensor) -> torch.Tensor:
    squeeze = x.dim() == 1
    if squeeze:
        x = x.unsqueeze(0)
    if x.dim() != 2:
        raise ValueError(f"expected 1-D or 2-D input, got shape {tuple(x.shape)}")
    n = x.shape[1]
    x = _rows2d(x, n)
    y = torch.empty_like(x, memory_format=torch.contiguous_format)
    lib = _lib.load()
    with torch.cuda.device(x.device):
        _lib.check(getattr(lib, fn_name)(_ptr(x), _ptr(y), x.shape[0], n, _ld(x, n), _ld(y, n), _stream(x)))
    return y[0] if squeeze else y


def dct(x: torch.Tensor) -> torch.Tensor:
    """Row-wise orthonormal DCT-II (transforms.py:137-145)."""
    return _transform("acdc_dct2_f32", x)


def idct(x: torch.Tensor) -> torch.Tensor:
    """Row-wise orthonormal DCT-III, the inverse of :func:`dct` (transforms.py:148-156)."""
    return _transform("acdc_dct3_f32", x)


def _fft_rows(z: torch.Tensor, inverse: bool, out: torch.Tensor | None = None) -> torch.Tensor:
    squeeze = z.dim() == 1
    if squeeze:
        z = z.unsqueeze(0)
    if not isinstance(z, torch.Tensor) or not z.is_cuda or z.dim() != 2:
        raise ValueError("expected a 1-D or 2-D CUDA tensor")
    if z.dtype != torch.complex64:
        z = z.to(torch.complex64)
    if z.stride(1) != 1 or (z.shape[0] > 1 and z.stride(0) < z.shape[1]):
        z = z.contiguous()
    n = z.shape[1]
    y = torch.empty_like(z, memory_format=torch.contiguous_format) if out is None else out
    lib = _lib.load()
    with torch.cuda.device(z.device):
        _lib.check(lib.acdc_fft_c64(_ptr(z), _ptr(y), z.shape[0], n, 1 if inverse else 0, _ld(z, n), _ld(y, n),
                                    _stream(z)))
    return y[0] if squeeze else y


def fft(z: torch.Tensor) -> torch.Tensor:
    """Unnormalised forward DFT of each complex64 row (transforms.py:166-171)."""
    return _fft_rows(z, False)


def ifft(z: torch.Tensor) -> torch.Tensor:
    """Inverse DFT of each complex64 row, scaled by 1/N (transforms.py:174-179)."""
    return _fft_rows(z, True)


class AcdcFunction(torch.autograd.Function):
    """Autograd wrapper: forward = acdc_fwd_cache_f32, which also keeps
    h2 = C2(a*x) like the reference's cache (layers.py:145), and backward =
    acdc_bwd_cached_f32 (the TMEM backward at 512 <= N <= 8192); sizes without
    an h2 cache recompute it (acdc_bwd_f32).  Parameter grads
    are returned (accumulate=False) and summed into ``.grad`` by autograd."""

    @staticmethod
    def forward(ctx, x, a, d, bias):
        n = a.shape[0]
        rows = x.shape[0] if x.dim() == 2 else 0
        hc = new_h2cache(rows, n, x.device) if (rows > 0 and h2cache_supported(n)) else None
        y = acdc_forward(x, a, d, bias, h2cache=hc)
        if hc is None:
            ctx.save_for_backward(x, a, d)
        else:
            ctx.save_for_backward(x, a, d, hc)
        return y

    @staticmethod
    def backward(ctx, gy):
        x, a, d, *hc = ctx.saved_tensors
        n = a.shape[0]
        ga = torch.empty(n, dtype=torch.float32, device=x.device)
        gd = torch.empty_like(ga)
        gb = torch.empty_like(ga)
        dx = acdc_backward(x, gy, a, d, ga, gd, gb, accumulate=False, h2cache=hc[0] if hc else None)
        return dx, ga, gd, gb


def acdc(x, a, d, bias):
    """Differentiable ACDC layer: ``AcdcFunction.apply``."""
    return AcdcFunction.apply(x, a, d, bias)


# ----------------------------------------------------------------- AFDF


def _crows2d(x: torch.Tensor, n: int, name: str = "x") -> torch.Tensor:
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if x.dim() != 2 or x.shape[1] != n:
        raise ValueError(f"{name} must have shape (batch, {n}), got {tuple(x.shape)}")
    if x.dtype != torch.complex64:
        x = x.to(torch.complex64)
    return x.contiguous()


def _cvec(v: torch.Tensor, n: int, dev, name: str) -> torch.Tensor:
    if v.dim() != 1 or v.shape[0] != n:
        raise ValueError(f"{name} must have shape ({n},), got {tuple(v.shape)}")
    return v.to(device=dev, dtype=torch.complex64).contiguous()


def afdf_forward(x: torch.Tensor, a: torch.Tensor, d: torch.Tensor, out=None) -> torch.Tensor:
    """y = IFFT(d * FFT(a * x)) row-wise, complex64 (layers.py:199-204)."""
    n = a.shape[0]
    x = _crows2d(x, n)
    a, d = _cvec(a, n, x.device, "a"), _cvec(d, n, x.device, "d")
    y = torch.empty_like(x) if out is None else _check_out(out, x)
    lib = _lib.load()
    with torch.cuda.device(x.device):
        _lib.check(lib.afdf_fwd_c64(_ptr(x), _ptr(y), _ptr(a), _ptr(d), x.shape[0], n, n, n, _stream(x)))
    return y


def afdf_backward(x, dy, a, d, grad_a, grad_d, accumulate: bool = True, out=None) -> torch.Tensor:
    """dx and (accumulated) complex diagonal gradients dL/dRe + i dL/dIm
    (layers.py:206-215).  grad_a / grad_d: complex64 (n,) CUDA tensors, in place."""
    n = a.shape[0]
    x = _crows2d(x, n)
    dy = _crows2d(dy, n, "grad_y")
    if dy.shape[0] != x.shape[0]:
        raise ValueError(f"grad_y has {dy.shape[0]} rows, input had {x.shape[0]}")
    dev = x.device
    a, d = _cvec(a, n, dev, "a"), _cvec(d, n, dev, "d")
    for g in (grad_a, grad_d):
        if g.device != dev or g.dtype != torch.complex64 or not g.is_contiguous() or g.shape != (n,):
            raise ValueError("gradient buffers must be contiguous complex64 (n,) tensors on the input device")
    dx = torch.empty_like(x) if out is None else _check_out(out, x)
    lib = _lib.load()
    with _on(dev):
        wsb = lib.afdf_bwd_workspace_bytes(x.shape[0], n)
        if wsb == 0:
            _lib.check(_lib.ACDC_E_SIZE if n > 16384 or n < 2 else _lib.ACDC_E_CUDA)
        ws = torch.empty((wsb + 3) // 4, dtype=torch.float32, device=dev)
        _lib.check(
            lib.afdf_bwd_c64(
                _ptr(x), _ptr(dy), _ptr(dx), _ptr(a), _ptr(d), _ptr(grad_a), _ptr(grad_d), 1 if accumulate else 0,
                _ptr(ws), wsb, x.shape[0], n, n, n, n, _stream(x),
            )
        )
    return dx


class AfdfFunction(torch.autograd.Function):
    """Autograd wrapper for the complex AFDF layer.  The kernels return
    dL/dRe + i dL/dIm, which is what torch's complex autograd propagates
    (conjugate Wirtinger convention)."""

    @staticmethod
    def forward(ctx, x, a, d):
        y = afdf_forward(x, a, d)
        ctx.save_for_backward(x, a, d)
        return y

    @staticmethod
    def backward(ctx, gy):
        x, a, d = ctx.saved_tensors
        n = a.shape[0]
        ga = torch.empty(n, dtype=torch.complex64, device=x.device)
        gd = torch.empty_like(ga)
        dx = afdf_backward(x, gy, a, d, ga, gd, accumulate=False)
        return dx, ga, gd


def afdf(x, a, d):
    """Differentiable AFDF layer: ``AfdfFunction.apply``."""
    return AfdfFunction.apply(x, a, d)


# ----------------------------------------------------------- fused cascade


def cascade_supported(n: int) -> bool:
    """Sizes of the fused cascade kernels (row-pair engine, h2 checkpoints)."""
    return 256 <= n <= 16384 and (n & (n - 1)) == 0


def cascade_hl_supported(n: int) -> bool:
    """Sizes where ACDC-only stacks run the half-length-plan fused cascade."""
    return cascade_supported(n) and _lib.load().cascade_hl_supported(int(n)) == 1


def cascade_forward(x: torch.Tensor, a: torch.Tensor, d: torch.Tensor, bias: torch.Tensor, perm: torch.Tensor | None,
                    flags: torch.Tensor, out=None, hl: bool = False):
    """Fused forward of ``depth`` blocks  x <- perm(relu(ACDC(x)))  (layers.py:336-339).

    a, d, bias: (depth, n) fp32; perm: (depth, n) int32 or None; flags: (depth,)
    uint8 (bit0 ReLU, bit1 permutation after the block).  Returns (y, ckpt)
    where ckpt holds the per-block checkpoints for :func:`cascade_backward`."""
    depth, n = a.shape
    x = _rows2d(x, n)
    dev = x.device
    a, d, bias = (v.to(device=dev, dtype=torch.float32).contiguous() for v in (a, d, bias))
    lib = _lib.load()
    if lib.cascade_ckpt_bytes(max(x.shape[0], 1), n, depth) == 0:
        raise ValueError(f"the fused cascade needs 256 <= n <= 16384, got {n}")
    nbytes = lib.cascade_ckpt_bytes(x.shape[0], n, depth)  # 0 for an empty batch
    ckpt = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    y = torch.empty_like(x, memory_format=torch.contiguous_format) if out is None else _check_out(out, x)
    if x.shape[0] == 0:
        return y, ckpt
    with _on(dev):
        if hl:  # ACDC-only stack on the half-length plan (x, y, params 16-byte aligned: _rows2d / contiguous)
            _lib.check(lib.cascade_fwd_hl_f32(_ptr(x), _ptr(y), depth, n, _ptr(a), _ptr(d), _ptr(bias), _ptr(ckpt),
                                              x.shape[0], _ld(x, n), _ld(y, n), _stream(x)))
        else:
            _lib.check(lib.cascade_fwd_f32(_ptr(x), _ptr(y), depth, n, _ptr(a), _ptr(d), _ptr(bias), _ptr(perm),
                                           _ptr(flags), _ptr(ckpt), x.shape[0], _ld(x, n), _ld(y, n), _stream(x)))
    return y, ckpt


def _ckpt_views(ckpt: torch.Tensor, rows: int, n: int, depth: int):
    xs = ckpt[: (depth - 1) * rows * n].view(depth - 1, rows, n) if depth > 1 else None
    per = ((rows + 1) // 2) * 2 * n
    base = (depth - 1) * rows * n
    h2 = [ckpt[base + l * per: base + (l + 1) * per] for l in range(depth)]
    return xs, h2


def cascade_backward(x: torch.Tensor, dy: torch.Tensor, a, d, perm: torch.Tensor | None, flags,
                     ckpt: torch.Tensor, grads, accumulate: bool = True, sgd=None, on_block=None,
                     perm_inv: torch.Tensor | None = None, hl: bool = False) -> torch.Tensor:
    """Backward of :func:`cascade_forward` (layers.py:341-344): one cached-h2
    block backward per block, last to first, each applying the previous block's
    ReLU mask and inverse permutation in its epilogue.  ``a``, ``d``: sequences
    of (n,) tensors per block; ``grads``: per block (grad_a, grad_d, grad_bias)
    fp32 (n,) tensors, accumulated in place; ``flags``: host list of ints.
    ``sgd``: optional per-block (params, velocities, lr3, wd3, momentum): each
    block's momentum-SGD step is fused into its gradient reduction
    (:func:`acdc_backward_sgd`); the grads are then added in and zeroed.
    ``on_block(l)`` is called after block l's kernels are enqueued (e.g. to
    start that block's gradient all-reduce while earlier blocks run).
    ``perm_inv`` (argsort of each perm row): where the TMEM backward runs, the
    permutation after block l is applied as a gather in block l's dy load
    instead of a scattered store in block l+1's epilogue."""
    depth = len(a)
    n = a[0].shape[0]
    x = _rows2d(x, n)
    g = _rows2d(dy, n, "grad_y")
    rows = x.shape[0]
    if g.shape[0] != rows:
        raise ValueError(f"grad_y has {g.shape[0]} rows, forward input had {rows}")
    dev = x.device
    if rows == 0:  # empty batch: gradients unchanged (+= 0), or zeroed without accumulate
        if not accumulate:
            for gr in grads:
                for t in gr:
                    t.zero_()
        if sgd is not None:
            for l in range(depth - 1, -1, -1):
                prm, vel, lr3, wd3, mu = sgd[l]
                acdc_backward_sgd(x, g, prm, vel, lr3, wd3, mu, grads=grads[l], accumulate=accumulate)
        return torch.empty_like(g)
    xs, h2 = _ckpt_views(ckpt, rows, n, depth)
    fl = [int(f) for f in flags]
    lib = _lib.load()
    if hl:  # checkpoints from cascade_fwd_hl_f32: every block is a plain single-layer cached backward
        return _cascade_backward_hl(x, g, a, d, xs, h2, grads, accumulate, sgd, on_block)
    gather = sgd is None and perm_inv is not None and lib.cascade_gather_supported(n) == 1
    # Without a per-block hook or fused SGD, every block writes only its
    # gradient partials and one launch reduces all blocks at the end: the
    # block-to-block chain no longer waits for a reduction per block.
    dstride = lib.cascade_defer_ws_bytes(rows, n) if (sgd is None and on_block is None) else 0
    tab = _grad_table(grads, dev) if dstride else None
    if tab is not None:
        return _cascade_backward_deferred(x, g, a, d, perm, fl, xs, h2, grads, tab, accumulate,
                                          perm_inv if gather else None, dstride)
    with _on(dev):
        wsb = lib.acdc_bwd_workspace_bytes(rows, n)
        ws = torch.empty((wsb + 3) // 4, dtype=torch.float32, device=dev)
        for l in range(depth - 1, -1, -1):
            if gather:  # relu mask in the epilogue, the permutation as this block's dy gather
                xl = x if l == 0 else xs[l - 1]
                prev = fl[l - 1] if l > 0 else 0
                gi = perm_inv[l] if (l < depth - 1 and fl[l] & 2) else None
                out = torch.empty_like(g)
                ga, gd, gb = grads[l]
                al, dl = _vec(a[l], n, dev, "a"), _vec(d[l], n, dev, "d")
                _lib.check(lib.cascade_bwd_block_gather_f32(
                    _ptr(xl), _ptr(g), _ptr(out), _ptr(al), _ptr(dl), _ptr(h2[l]), _ptr(gi), 1 if prev & 1 else 0,
                    _ptr(ga), _ptr(gd), _ptr(gb), 1 if accumulate else 0, _ptr(ws), wsb, rows, n, _ld(xl, n),
                    _ld(g, n), n, _stream(x)))
                g = out
                if on_block is not None:
                    on_block(l)
                continue
            xl = x if l == 0 else xs[l - 1]
            prev = fl[l - 1] if l > 0 else 0
            pp = perm[l - 1] if (l > 0 and prev & 2) else None
            out = torch.empty_like(g)
            ga, gd, gb = grads[l]
            if sgd is not None:
                prm, vel, lr3, wd3, mu = sgd[l]
                acdc_backward_sgd(xl, g, prm, vel, lr3, wd3, mu, grads=(ga, gd, gb), accumulate=accumulate, out=out,
                                  h2cache=h2[l], prev_perm=pp, prev_relu=bool(prev & 1), ws=ws, h2_rowpair=True)
                g = out
                if on_block is not None:
                    on_block(l)
                continue
            al, dl = _vec(a[l], n, dev, "a"), _vec(d[l], n, dev, "d")
            _lib.check(lib.cascade_bwd_block_f32(
                _ptr(xl), _ptr(g), _ptr(out), _ptr(al), _ptr(dl), _ptr(h2[l]), _ptr(pp), 1 if prev & 1 else 0,
                _ptr(ga), _ptr(gd), _ptr(gb), 1 if accumulate else 0, _ptr(ws), wsb, rows, n, _ld(xl, n), _ld(g, n),
                n, _stream(x)))
            g = out
            if on_block is not None:
                on_block(l)
    return g


def _cascade_backward_hl(x, g, a, d, xs, h2, grads, accumulate, sgd, on_block):
    """Backward of the half-length-plan cascade (ACDC-only blocks): deferred
    block partials + one multi-block reduction, or (per-block hook / fused
    SGD) the single-layer cached backward per block."""
    depth = len(a)
    n = a[0].shape[0]
    rows = x.shape[0]
    dev = x.device
    lib = _lib.load()
    stride = lib.cascade_hl_defer_ws_bytes(rows, n) if (sgd is None and on_block is None) else 0
    tab = _grad_table(grads, dev) if stride else None
    with _on(dev):
        if tab is not None:
            if any(t.shape != (n,) for gr in grads for t in gr):
                raise ValueError("gradient buffers must be contiguous fp32 (n,) tensors on the input device")
            ws = torch.empty(depth * stride // 4, dtype=torch.float32, device=dev)
            for l in range(depth - 1, -1, -1):
                xl = x if l == 0 else xs[l - 1]
                out = torch.empty_like(g)
                al, dl = _vec(a[l], n, dev, "a"), _vec(d[l], n, dev, "d")
                _lib.check(lib.cascade_bwd_hl_defer_f32(
                    _ptr(xl), _ptr(g), _ptr(out), _ptr(al), _ptr(dl), _ptr(h2[l]), ws.data_ptr() + l * stride,
                    stride, rows, n, _ld(xl, n), _ld(g, n), n, _stream(x)))
                g = out
            _lib.check(lib.cascade_grad_reduce_hl_f32(_ptr(ws), stride, depth, rows, n, _ptr(tab),
                                                      1 if accumulate else 0, _stream(x)))
            return g
        for l in range(depth - 1, -1, -1):
            xl = x if l == 0 else xs[l - 1]
            if sgd is not None:
                prm, vel, lr3, wd3, mu = sgd[l]
                g = acdc_backward_sgd(xl, g, prm, vel, lr3, wd3, mu, grads=grads[l], accumulate=accumulate,
                                      h2cache=h2[l])
            else:
                ga, gd, gb = grads[l]
                g = acdc_backward(xl, g, a[l], d[l], ga, gd, gb, accumulate=accumulate, h2cache=h2[l])
            if on_block is not None:
                on_block(l)
    return g


_grad_tables: dict = {}


def _grad_table(grads, dev) -> torch.Tensor:
    """Device array of the blocks' (grad_a, grad_d, grad_bias) pointers, cached
    per pointer tuple (the layers' gradient buffers are persistent)."""
    for gr in grads:
        for t in gr:
            if t.device != dev or t.dtype != torch.float32 or not t.is_contiguous() or t.dim() != 1:
                raise ValueError("gradient buffers must be contiguous fp32 (n,) tensors on the input device")
    key = (dev.index, tuple(t.data_ptr() for gr in grads for t in gr))
    tab = _grad_tables.get(key)
    if tab is None:
        if torch.cuda.is_current_stream_capturing():
            return None  # no host-to-device copy inside a capture: the caller uses the per-block reductions
        if len(_grad_tables) > 64:
            _grad_tables.clear()
        tab = torch.tensor(key[1], dtype=torch.int64).to(dev)
        _grad_tables[key] = tab
    return tab


def _cascade_backward_deferred(x, g, a, d, perm, fl, xs, h2, grads, tab, accumulate, perm_inv, stride):
    depth = len(a)
    n = a[0].shape[0]
    rows = x.shape[0]
    dev = x.device
    lib = _lib.load()
    if any(t.shape != (n,) for gr in grads for t in gr):
        raise ValueError("gradient buffers must be contiguous fp32 (n,) tensors on the input device")
    has_perm = any(f & 2 for f in fl[:-1])
    pairs = (os.environ.get("ACDC_CASCADE_PAIR", "1") != "0" and depth >= 2 and (perm_inv is not None or not has_perm)
             and lib.cascade_pair_supported(rows, n) == 1)
    with _on(dev):
        ws = torch.empty(depth * stride // 4, dtype=torch.float32, device=dev)
        l = depth - 1
        while pairs and l >= 1:  # blocks l (hi) and l-1 (lo) in one launch, the dx between them on chip
            hi, lo = l, l - 1
            xh = xs[hi - 1]
            xlo = x if lo == 0 else xs[lo - 1]
            gh = perm_inv[hi] if (perm_inv is not None and hi < depth - 1 and fl[hi] & 2) else None
            gl = perm_inv[lo] if (perm_inv is not None and fl[lo] & 2) else None
            out = torch.empty_like(g)
            ah, dh = _vec(a[hi], n, dev, "a"), _vec(d[hi], n, dev, "d")
            al, dl = _vec(a[lo], n, dev, "a"), _vec(d[lo], n, dev, "d")
            _lib.check(lib.cascade_bwd_pair_defer_f32(
                _ptr(xh), _ptr(xlo), _ptr(g), _ptr(out), _ptr(ah), _ptr(dh), _ptr(al), _ptr(dl), _ptr(h2[hi]),
                _ptr(h2[lo]), _ptr(gh), _ptr(gl), 1 if fl[lo] & 1 else 0, 1 if (lo > 0 and fl[lo - 1] & 1) else 0,
                ws.data_ptr() + hi * stride, ws.data_ptr() + lo * stride, stride, rows, n, _ld(xh, n),
                _ld(xlo, n), _ld(g, n), n, _stream(x)))
            g = out
            l -= 2
        for l in range(l, -1, -1):
            xl = x if l == 0 else xs[l - 1]
            prev = fl[l - 1] if l > 0 else 0
            if perm_inv is not None:  # the permutation after block l as this block's dy gather
                pp, gi = None, (perm_inv[l] if (l < depth - 1 and fl[l] & 2) else None)
            else:  # the permutation before block l as a scatter in its epilogue
                pp, gi = (perm[l - 1] if (l > 0 and prev & 2) else None), None
            out = torch.empty_like(g)
            al, dl = _vec(a[l], n, dev, "a"), _vec(d[l], n, dev, "d")
            _lib.check(lib.cascade_bwd_block_defer_f32(
                _ptr(xl), _ptr(g), _ptr(out), _ptr(al), _ptr(dl), _ptr(h2[l]), _ptr(pp), _ptr(gi),
                1 if prev & 1 else 0, ws.data_ptr() + l * stride, stride, rows, n, _ld(xl, n), _ld(g, n), n,
                _stream(x)))
            g = out
        _lib.check(lib.cascade_grad_reduce_f32(_ptr(ws), stride, depth, rows, n, _ptr(tab), 1 if accumulate else 0,
                                               _stream(x)))
    return g


# ------------------------------------------------- host-buffer pipelined step


class HostPipeline:
    """Forward + backward of one ACDC layer on HOST (pinned) buffers, with the
    batch split into chunks so host->device copies, kernels and device->host
    copies of different chunks overlap on three streams (PCIe is full duplex).

    ``step(x_host, dy_host, y_host, dx_host)`` computes y = layer(x) and dx,
    writes them back to host, and accumulates the parameter gradients into
    ``grads`` (device, summed over all chunks: the reference's "+=" semantics).
    Chunks are independent rows, so the result equals one full-batch call.

    ``direct_out``: the kernels store y and dx straight into the pinned host
    buffers (mapped through unified addressing: posted PCIe writes from the
    SMs), so there is no device->host copy stage to schedule around.

    ``overlap_steps``: a step's uploads wait only for their device buffers,
    not for the caller's stream, so they overlap the previous step's last
    downloads (the kernels still follow the caller's stream: parameters and
    gradients).  The host inputs must not be rewritten until the step's
    uploads have completed, as with any asynchronous copy.
    """

    def __init__(self, n: int, rows: int, device, chunks: int = 8, h2cache: bool = True, nbuf: int = 2,
                 ramp: bool = False, direct_out: bool = False, overlap_steps: bool = True):
        self.n, self.rows, self.dev = n, rows, torch.device(device)
        self.overlap_steps = overlap_steps
        self.direct_out = direct_out
        self.spans = self.plan(rows, chunks, ramp)
        self.chunks = len(self.spans)
        mx = max(b - a for a, b in self.spans)
        # nbuf device buffer sets: chunk i+1.. upload while chunk i computes / downloads
        self.nbuf = max(2, nbuf)
        self.xd = [torch.empty(mx, n, device=self.dev) for _ in range(self.nbuf)]
        self.dyd = [torch.empty(mx, n, device=self.dev) for _ in range(self.nbuf)]
        nout = 0 if direct_out else self.nbuf
        self.yd = [torch.empty(mx, n, device=self.dev) for _ in range(nout)]
        self.dxd = [torch.empty(mx, n, device=self.dev) for _ in range(nout)]
        self.hc = ([new_h2cache(mx, n, self.dev) for _ in range(self.nbuf)]
                   if (h2cache and h2cache_supported(n)) else None)
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_cmp = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        # last compute / download that used each buffer set, across steps: the next
        # step's uploads only wait for these, so they overlap this step's downloads
        self._buf_done = [None] * self.nbuf
        self._buf_down = [None] * self.nbuf
        prepare(n, self.dev)

    @staticmethod
    def plan(rows: int, chunks: int, ramp: bool = True):
        """Row spans.  With ``ramp`` the first and last chunks shrink
        geometrically (1/8, 1/4, 1/2 of the uniform size): the upload of the
        first chunk and the download of the last one are the only transfers
        that cannot overlap a transfer in the other direction."""
        chunks = max(1, min(chunks, rows))
        u = -(-rows // chunks)
        sizes = []
        if ramp and chunks >= 4 and u >= 16:
            head = [max(1, u // 8), max(1, u // 4), max(1, u // 2)]
            tail = head[::-1]
            mid = rows - sum(head) - sum(tail)
            if mid > 0:
                k = max(1, -(-mid // u))
                base, extra = divmod(mid, k)
                sizes = head + [base + (1 if i < extra else 0) for i in range(k)] + tail
        if not sizes:
            base, extra = divmod(rows, chunks)
            sizes = [base + (1 if i < extra else 0) for i in range(chunks)]
        # interior boundaries even: the kernels pack rows (2k, 2k+1) into one
        # complex FFT, so even chunk starts keep the full-batch pairing and
        # y / dx bit-identical to one call over all rows
        bounds, lo = [0], 0
        for m in sizes:
            lo += m
            b = rows if lo >= rows else lo & ~1
            if b > bounds[-1]:
                bounds.append(b)
        if bounds[-1] != rows:
            bounds.append(rows)
        return [(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1)]

    def step(self, x_host, dy_host, y_host, dx_host, a, d, bias, grads, accumulate=True, timeline=False):
        """All host tensors must be pinned CPU fp32 (rows, n).  Returns after
        enqueueing; call ``torch.cuda.synchronize()`` (or an event) to wait."""
        ga, gd, gb = grads
        up = [torch.cuda.Event(enable_timing=timeline) for _ in self.spans]
        done = [torch.cuda.Event(enable_timing=timeline) for _ in self.spans]
        down = [torch.cuda.Event(enable_timing=timeline) for _ in self.spans]
        cur = torch.cuda.current_stream(self.dev)
        # the kernels and downloads follow the caller's stream (parameters, gradients);
        # the uploads only need their buffer set free (previous step included)
        for s in (self.s_cmp, self.s_out) if self.overlap_steps else (self.s_in, self.s_cmp, self.s_out):
            s.wait_stream(cur)
        if not accumulate:
            with torch.cuda.stream(self.s_cmp):
                ga.zero_()
                gd.zero_()
                gb.zero_()
        nb = self.nbuf
        for i, (lo, hi) in enumerate(self.spans):
            k, m = i % nb, hi - lo
            with torch.cuda.stream(self.s_in):
                prev = done[i - nb] if i >= nb else self._buf_done[k]
                if prev is not None:  # buffer set k is free once its previous chunk was computed
                    self.s_in.wait_event(prev)
                self.xd[k][:m].copy_(x_host[lo:hi], non_blocking=True)
                self.dyd[k][:m].copy_(dy_host[lo:hi], non_blocking=True)
                up[i].record(self.s_in)
            with torch.cuda.stream(self.s_cmp):
                self.s_cmp.wait_event(up[i])
                if not self.direct_out:  # outputs of the buffer's previous chunk must be downloaded first
                    prev = down[i - nb] if i >= nb else self._buf_down[k]
                    if prev is not None:
                        self.s_cmp.wait_event(prev)
                hc = self.hc[k] if self.hc is not None else None
                yo = y_host[lo:hi] if self.direct_out else self.yd[k][:m]
                dxo = dx_host[lo:hi] if self.direct_out else self.dxd[k][:m]
                acdc_forward(self.xd[k][:m], a, d, bias, out=yo, h2cache=hc)
                acdc_backward(self.xd[k][:m], self.dyd[k][:m], a, d, ga, gd, gb, accumulate=True, out=dxo,
                              h2cache=hc)
                done[i].record(self.s_cmp)
            if self.direct_out:
                down[i] = done[i]
                continue
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(done[i])
                y_host[lo:hi].copy_(self.yd[k][:m], non_blocking=True)
                dx_host[lo:hi].copy_(self.dxd[k][:m], non_blocking=True)
                down[i].record(self.s_out)
        for i in range(max(0, len(self.spans) - nb), len(self.spans)):
            self._buf_done[i % nb] = done[i]
            self._buf_down[i % nb] = down[i]
        for s in (self.s_in, self.s_cmp, self.s_out):
            cur.wait_stream(s)
        if timeline:  # (upload, compute, download) completion events per chunk
            return list(zip(up, done, down))


# ------------------------------------------------- ReLU / permutation layers


def relu_forward(x: torch.Tensor) -> torch.Tensor:
    """y = x > 0 ? x : 0 (layers.py:225-229), native kernel."""
    x = _rows2d(x, x.shape[1])
    y = torch.empty_like(x, memory_format=torch.contiguous_format)
    with torch.cuda.device(x.device):
        _lib.check(_lib.load().acdc_relu_fwd_f32(_ptr(x), _ptr(y), x.shape[0], x.shape[1], _ld(x, x.shape[1]),
                                                 x.shape[1], _stream(x)))
    return y


def relu_backward(y: torch.Tensor, dy: torch.Tensor) -> torch.Tensor:
    """dx = y > 0 ? dy : 0 with y the forward output (layers.py:231-233)."""
    n = y.shape[1]
    y, dy = _rows2d(y, n, "y"), _rows2d(dy, n, "grad_y")
    if dy.shape != y.shape:
        raise ValueError(f"grad_y has shape {tuple(dy.shape)}, the forward output {tuple(y.shape)}")
    dx = torch.empty_like(dy, memory_format=torch.contiguous_format)
    with torch.cuda.device(y.device):
        _lib.check(_lib.load().acdc_relu_bwd_f32(_ptr(y), _ptr(dy), _ptr(dx), y.shape[0], n, _ld(y, n), _ld(dy, n),
                                                 n, _stream(y)))
    return dx


def gather_cols(x: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """y[:, j] = x[:, idx[j]] for fp32 or complex64 rows (idx int32 on the device)."""
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dim() != 2:
        raise ValueError("expected a 2-D CUDA tensor")
    if x.dtype not in (torch.float32, torch.complex64):
        x = x.to(torch.complex64 if x.is_complex() else torch.float32)
    if x.stride(1) != 1 or (x.shape[0] > 1 and x.stride(0) < x.shape[1]):
        x = x.contiguous()
    n = x.shape[1]
    y = torch.empty_like(x, memory_format=torch.contiguous_format)
    with torch.cuda.device(x.device):
        _lib.check(_lib.load().acdc_gather_cols(_ptr(x), _ptr(y), _ptr(idx), x.shape[0], n, x.element_size(),
                                                _ld(x, n), n, _stream(x)))
    return y
