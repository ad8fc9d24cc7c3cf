"""Kernel-plugin module for the reference's secondary seam (``backend.py:30-42``).

``acdc.backend.get_kernels(name)`` returns a module exposing ``COMPILED`` and
three functions on host numpy arrays (``_kernels.pyx:18-91``):

    fft_inplace(z, rev, tw, inverse)             z: complex128 (B, N), in place
    dct2_batch(x, out, reorder, rev, tw, w4s)    x, out: float64 (B, N)
    dct3_batch(y, out, reorder, rev, tw, u1, u2) y, out: float64 (B, N)

This module has the same names, argument meaning and in-place / caller-owned
output behaviour, computed by the B200 kernels through the C ABI
(``acdc_fft_c64``, ``acdc_dct2_f32``, ``acdc_dct3_f32``): each call rounds the
rows to fp32 / complex64, copies them to the GPU, transforms them and writes
the result back into the caller's fp64 array.  The table arguments (bit
reversal, twiddles, Makhoul factors) are accepted for signature compatibility;
the device kernels use their own fp64-built tables of the same values.  It is
the numerics seam (the reference's transform checks through GPU transforms),
not the fast path: the layer API keeps data on the device.

A maintainer wires it in with one branch in ``get_kernels``.
There is no CPU fallback: without the CUDA library every call raises.
"""

from __future__ import annotations

import numpy as np
import torch

from . import functional as F

COMPILED = True

__all__ = ["COMPILED", "fft_inplace", "dct2_batch", "dct3_batch"]


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("the b200 kernel backend needs a CUDA device")
    return torch.device("cuda", torch.cuda.current_device())


def _rows(a: np.ndarray, name: str) -> np.ndarray:
    if a.ndim != 2:
        raise ValueError(f"{name} must be a 2-D (batch, n) array, got shape {a.shape}")
    return a


def fft_inplace(z, rev, tw, inverse):
    """In-place batched DFT of the rows of ``z`` (complex128, (B, N));
    ``inverse`` scales by 1/N (``_kernels.pyx:49-57``)."""
    z = _rows(z, "z")
    if z.shape[1] == 0 or z.shape[0] == 0:
        return
    dev = _device()
    zd = torch.from_numpy(np.ascontiguousarray(z, dtype=np.complex64)).to(dev)
    F._fft_rows(zd, bool(inverse), out=zd)
    z[...] = zd.cpu().numpy()


def dct2_batch(x, out, reorder, rev, tw, w4s):
    """Orthonormal DCT-II of each row of ``x`` into ``out`` (``_kernels.pyx:60-73``)."""
    x = _rows(x, "x")
    if x.shape[0] == 0:
        return
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(_device())
    out[...] = F.dct(xd).cpu().numpy()


def dct3_batch(y, out, reorder, rev, tw, u1, u2):
    """Orthonormal DCT-III of each row of ``y`` into ``out`` (``_kernels.pyx:76-91``)."""
    y = _rows(y, "y")
    if y.shape[0] == 0:
        return
    yd = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float32)).to(_device())
    out[...] = F.idct(yd).cpu().numpy()
