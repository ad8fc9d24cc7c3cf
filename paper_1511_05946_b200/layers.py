"""Drop-in mirror of the reference layer API (``acdc.layers``) on B200 kernels.

Same constructors, methods, attribute names and error behaviour as
``/root/reference/pkg/src/acdc/layers.py``; the numerics run through the
sm_100a kernels (``functional.py`` -> ``libacdc_b200.so``), in fp32.

* Inputs may be CUDA tensors (kept on device; the result is a CUDA tensor) or
  host arrays / tensors (copied to the layer's device; the result comes back
  as a float64 numpy array, like the reference).
* Parameters (``a``, ``d``, ``bias_d``) and gradient accumulators are fixed
  CUDA fp32 storage updated in place (layers.py:14-15); ``backward``
  accumulates into the gradients (layers.py:152-155) until ``zero_grads``.
* ``backward`` before ``forward`` raises ``RuntimeError`` and consumes the
  cache unless ``retain_cache`` (layers.py:99-105).
* Like the reference (layers.py:145), ``AcdcLayer`` caches ``x`` and
  ``h2 = C2(a * x)`` (in the kernels' native layout) on the sizes that support
  it (256 <= N <= 16384); elsewhere, or with ``cache_h2=False``, the backward
  kernel recomputes h2.
* ``save_cascade`` / ``load_cascade`` read and write the reference's JSON
  format (layers.py:466-554, format version 1).
"""

from __future__ import annotations

import json

from dataclasses import dataclass

import numpy as np
import torch

from . import functional as F
from .plans import DctPlan, FftPlan

__all__ = [
    "Param",
    "Layer",
    "AcdcLayer",
    "AfdfLayer",
    "ReluLayer",
    "PermutationLayer",
    "DenseLayer",
    "Cascade",
    "acdc_cascade",
    "afdf_cascade",
    "count_params",
    "save_cascade",
    "load_cascade",
    "FORMAT_VERSION",
]

FORMAT_VERSION = 1  # layers.py:47


def _is_pow2(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


def _device(device) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("the b200 backend needs a CUDA device (there is no CPU fallback)")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


@dataclass
class Param:
    """One trainable tensor plus its gradient accumulator (layers.py:50-63)."""

    name: str
    value: torch.Tensor
    grad: torch.Tensor
    decay: bool = False
    lr_mult: float = 1.0


class Layer:
    """Common interface: forward, backward, parameter access (layers.py:66-105)."""

    linear = True
    complex_domain = False
    n_in: int
    n_out: int
    device: torch.device

    def forward(self, x):
        raise NotImplementedError

    def backward(self, grad_y, retain_cache=False):
        raise NotImplementedError

    def params(self):
        return []

    def param_count(self):
        return 0

    def zero_grads(self):
        for p in self.params():
            p.grad.zero_()

    # -- input handling (layers.py:91-97): 2-D (batch, n_in) or ValueError
    def _check_input(self, x, dtype=torch.float32):
        host = not (isinstance(x, torch.Tensor) and x.is_cuda)
        if isinstance(x, torch.Tensor):
            t = x
        else:
            t = torch.as_tensor(np.asarray(x))
        if t.dim() != 2 or t.shape[1] != self.n_in:
            raise ValueError(
                f"{type(self).__name__} expects (batch, {self.n_in}) input, got shape {tuple(t.shape)}"
            )
        if host:
            t = t.to(dtype=dtype).pin_memory().to(self.device, non_blocking=True) if t.numel() else t.to(
                self.device, dtype=dtype)
        elif t.dtype != dtype or t.device != self.device:
            t = t.to(device=self.device, dtype=dtype)
        return t.contiguous(), host

    def _take_cache(self, retain):
        if getattr(self, "_cache", None) is None:
            raise RuntimeError(f"{type(self).__name__}.backward called before forward")
        cache = self._cache
        if not retain:
            self._cache = None
        return cache

    @staticmethod
    def _out(y: torch.Tensor, host: bool):
        if not host:
            return y
        dt = torch.complex128 if y.is_complex() else torch.float64
        return y.detach().to("cpu", dtype=dt).numpy()


class AcdcLayer(Layer):
    """Diagonal, DCT, diagonal-with-bias, inverse DCT (layers.py:108-156).

    ``dct_mode="fast"`` (power-of-two n) runs the fused sm_100a kernels.
    ``dct_mode="naive"`` is the reference's cosine-matrix mode
    (transforms.py:141, 152): any n >= 1, the transforms as dense fp32 GEMMs
    with the explicit DCT matrix on the device (cuBLAS; O(N^2), not the hot
    path).  ``backend`` takes the reference values ("auto", "compiled",
    "python", env ``ACDC_KERNEL_BACKEND``) plus "b200"; all select the B200
    kernels (``dct_plan.backend``).  ``dct_plan`` carries the reference
    plan's tables (``plans.DctPlan``).
    """

    def __init__(self, n, dct_mode="fast", backend="auto", device=None, cache_h2=True):
        self.dct_plan = DctPlan(n, mode=dct_mode, backend=backend)
        self.n_in = self.n_out = n
        self.dct_mode = dct_mode
        self.backend = backend
        self.naive = dct_mode == "naive"
        self.cache_h2 = bool(cache_h2) and not self.naive and F.h2cache_supported(n)
        self.device = _device(device)
        kw = dict(dtype=torch.float32, device=self.device)
        self.a = torch.ones(n, **kw)
        self.d = torch.ones(n, **kw)
        self.bias_d = torch.zeros(n, **kw)
        self.grad_a = torch.zeros(n, **kw)
        self.grad_d = torch.zeros(n, **kw)
        self.grad_bias_d = torch.zeros(n, **kw)
        self._params = [
            Param("a", self.a, self.grad_a),
            Param("d", self.d, self.grad_d),
            Param("bias_d", self.bias_d, self.grad_bias_d),
        ]
        self._cache = None
        if not self.naive:
            F.prepare(n, self.device)

    @property
    def n(self):
        return self.n_in

    def params(self):
        return self._params

    def param_count(self):
        return 3 * self.n_in

    def forward(self, x):
        x, host = self._check_input(x)
        if self.naive:  # h2 = (x a) C, y = (h2 d + b) C^T  (transforms.py:141, 152)
            C = self.dct_plan.cos_device(self.device)
            h2 = (x * self.a) @ C
            y = torch.addcmul(self.bias_d, h2, self.d) @ C.t()
            self._cache = (x, h2)
            return self._out(y, host)
        hc = F.new_h2cache(x.shape[0], self.n_in, self.device) if (self.cache_h2 and x.shape[0]) else None
        y = F.acdc_forward(x, self.a, self.d, self.bias_d, h2cache=hc)
        self._cache = (x, hc)
        return self._out(y, host)

    def backward(self, grad_y, retain_cache=False):
        x, hc = self._take_cache(retain_cache)
        gy, host = self._check_input(grad_y)
        if gy.shape[0] != x.shape[0]:
            raise ValueError(f"grad_y has {gy.shape[0]} rows, forward input had {x.shape[0]}")
        if self.naive:  # layers.py:148-156 with the dense transforms
            C = self.dct_plan.cos_device(self.device)
            g3 = gy @ C
            self.grad_bias_d += g3.sum(0)
            self.grad_d += (hc * g3).sum(0)
            g1 = (g3 * self.d) @ C.t()
            self.grad_a += (x * g1).sum(0)
            return self._out(g1 * self.a, host)
        dx = F.acdc_backward(x, gy, self.a, self.d, self.grad_a, self.grad_d, self.grad_bias_d, accumulate=True,
                             h2cache=hc)
        return self._out(dx, host)


class AfdfLayer(Layer):
    """Complex diagonals around the FFT pair, no bias (layers.py:159-215).

    Gradients are dL/dRe + i dL/dIm (layers.py:162-164).  ``fix_a`` removes
    ``a`` from ``params()`` (its gradient is still computed, layers.py:192-194,
    214); ``param_count`` stays 4N (layers.py:196-197).
    """

    linear = True
    complex_domain = True

    def __init__(self, n, backend="auto", fix_a=False, device=None):
        self.fft_plan = FftPlan(n, backend=backend)  # transforms.py:69-83 (raises for non-powers of two)
        self.n_in = self.n_out = n
        self.backend = backend
        self.fix_a = fix_a
        self.device = _device(device)
        kw = dict(dtype=torch.complex64, device=self.device)
        self.a = torch.ones(n, **kw)
        self.d = torch.ones(n, **kw)
        self.grad_a = torch.zeros(n, **kw)
        self.grad_d = torch.zeros(n, **kw)
        self._params = [Param("a", self.a, self.grad_a), Param("d", self.d, self.grad_d)]
        self._cache = None
        F.prepare(n, self.device)

    @property
    def n(self):
        return self.n_in

    def params(self):
        return self._params[1:] if self.fix_a else self._params

    def param_count(self):
        return 4 * self.n_in

    def _out(self, y, host):
        if not host:
            return y
        return y.detach().to("cpu", dtype=torch.complex128).numpy()

    def forward(self, x):
        x, host = self._check_input(x, torch.complex64)
        y = F.afdf_forward(x, self.a, self.d)
        self._cache = x
        return self._out(y, host)

    def backward(self, grad_y, retain_cache=False):
        x = self._take_cache(retain_cache)
        gy, host = self._check_input(grad_y, torch.complex64)
        if gy.shape[0] != x.shape[0]:
            raise ValueError(f"grad_y has {gy.shape[0]} rows, forward input had {x.shape[0]}")
        dx = F.afdf_backward(x, gy, self.a, self.d, self.grad_a, self.grad_d, accumulate=True)
        return self._out(dx, host)


class ReluLayer(Layer):
    """max(x, 0) with the strict ``x > 0`` mask (layers.py:218-233)."""

    linear = False

    def __init__(self, n, device=None):
        self.n_in = self.n_out = n
        self.device = _device(device)
        self._cache = None

    def forward(self, x):
        x, host = self._check_input(x)
        y = F.relu_forward(x)
        self._cache = y  # y > 0 exactly where x > 0: the strict mask
        return self._out(y, host)

    def backward(self, grad_y, retain_cache=False):
        y = self._take_cache(retain_cache)
        gy, host = self._check_input(grad_y)
        return self._out(F.relu_backward(y, gy), host)


class PermutationLayer(Layer):
    """Fixed permutation of the feature axis (layers.py:236-265)."""

    def __init__(self, n, perm=None, rng=None, device=None):
        self.n_in = self.n_out = n
        self.device = _device(device)
        if perm is None:
            if rng is None:
                raise ValueError("PermutationLayer needs an explicit perm or an rng")
            perm = rng.permutation(n)
        perm = np.asarray(perm.cpu() if isinstance(perm, torch.Tensor) else perm, dtype=np.int64)
        if sorted(perm.tolist()) != list(range(n)):
            raise ValueError("perm is not a bijection on 0..n-1")
        self.perm = perm
        self.inverse_perm = np.argsort(perm)
        self._perm_t = torch.as_tensor(perm, dtype=torch.int32, device=self.device)
        self._inv_t = torch.as_tensor(self.inverse_perm, dtype=torch.int32, device=self.device)
        self._cache = None

    @staticmethod
    def _dtype(x):
        """Dtype-agnostic like the reference (no cast): complex stays complex."""
        cplx = x.is_complex() if isinstance(x, torch.Tensor) else np.iscomplexobj(x)
        return torch.complex64 if cplx else torch.float32

    def forward(self, x):
        shape = tuple(x.shape) if hasattr(x, "shape") else np.shape(x)
        if shape[1:] != (self.n_in,):
            raise ValueError(f"PermutationLayer expects (batch, {self.n_in}) input")
        x, host = self._check_input(x, self._dtype(x))
        self._cache = True
        return self._out(F.gather_cols(x, self._perm_t), host)

    def backward(self, grad_y, retain_cache=False):
        self._take_cache(retain_cache)
        gy, host = self._check_input(grad_y, self._dtype(grad_y))
        return self._out(F.gather_cols(gy, self._inv_t), host)


class DenseLayer(Layer):
    """Dense y = xW + b baseline (layers.py:268-306), via cuBLAS (comparator only)."""

    def __init__(self, n_in, n_out, rng=None, device=None):
        self.n_in, self.n_out = n_in, n_out
        self.device = _device(device)
        kw = dict(dtype=torch.float32, device=self.device)
        if rng is not None:
            bound = np.sqrt(6.0 / (n_in + n_out))
            self.w = torch.as_tensor(rng.uniform(n_in, n_out, -bound, bound), **kw)
        else:
            self.w = torch.zeros(n_in, n_out, **kw)
        self.b = torch.zeros(n_out, **kw)
        self.grad_w = torch.zeros(n_in, n_out, **kw)
        self.grad_b = torch.zeros(n_out, **kw)
        self._params = [Param("w", self.w, self.grad_w, decay=True), Param("b", self.b, self.grad_b)]
        self._cache = None

    def params(self):
        return self._params

    def param_count(self):
        return self.n_in * self.n_out + self.n_out

    def forward(self, x):
        x, host = self._check_input(x)
        self._cache = x
        return self._out(torch.addmm(self.b, x, self.w), host)

    def backward(self, grad_y, retain_cache=False):
        x = self._take_cache(retain_cache)
        if isinstance(grad_y, torch.Tensor) and grad_y.is_cuda:
            gy, host = grad_y.to(torch.float32), False
        else:
            gy, host = torch.as_tensor(np.asarray(grad_y), dtype=torch.float32).to(self.device), True
        if tuple(gy.shape) != (x.shape[0], self.n_out):
            raise ValueError(f"gradient shape {tuple(gy.shape)} does not match output")
        self.grad_w.addmm_(x.t(), gy)
        self.grad_b.add_(gy.sum(0))
        return self._out(gy @ self.w.t(), host)


class Cascade:
    """Ordered layer stack with a unified forward/backward contract (layers.py:309-357)."""

    def __init__(self, layers):
        layers = list(layers)
        if not layers:
            raise ValueError("cascade needs at least one layer")
        for prev, nxt in zip(layers, layers[1:]):
            if prev.n_out != nxt.n_in:
                raise ValueError(
                    f"adjacent sizes differ: {type(prev).__name__} outputs {prev.n_out}, "
                    f"{type(nxt).__name__} expects {nxt.n_in}"
                )
        domains = {l.complex_domain for l in layers if not isinstance(l, PermutationLayer)}
        if len(domains) > 1:
            raise ValueError("cannot mix complex and real layers in one cascade")
        self.layers = layers
        self.complex_domain = any(l.complex_domain for l in layers)
        self._fused = self._fusion_plan(layers)
        self._cache = None

    @staticmethod
    def _fusion_plan(layers):
        """Blocks (ACDC [, ReLU] [, Perm]) covering the whole stack, ending in an
        ACDC layer, at a size the fused cascade kernels support; else None."""
        if not layers or not isinstance(layers[-1], AcdcLayer):
            return None
        n = layers[0].n_in
        if not F.cascade_supported(n) or any(l.n_in != n for l in layers):
            return None
        blocks, i = [], 0
        while i < len(layers):
            if not isinstance(layers[i], AcdcLayer) or layers[i].naive:
                return None
            blk = [layers[i], None, None]
            i += 1
            if i < len(layers) and isinstance(layers[i], ReluLayer):
                blk[1] = layers[i]
                i += 1
            if i < len(layers) and isinstance(layers[i], PermutationLayer):
                blk[2] = layers[i]
                i += 1
            blocks.append(blk)
        dev = blocks[0][0].device
        if any(b[0].device != dev for b in blocks):
            return None
        flags = [(1 if b[1] is not None else 0) | (2 if b[2] is not None else 0) for b in blocks]
        perm = perm_inv = None
        if any(f & 2 for f in flags):
            rows = [torch.as_tensor(b[2].perm if b[2] is not None else np.arange(n), dtype=torch.int32) for b in blocks]
            perm = torch.stack(rows).to(dev).contiguous()
            perm_inv = torch.argsort(perm.long(), dim=1).to(torch.int32).contiguous()
        # ACDC-only stacks (the reference's acdc_cascade) at the half-length plan's sizes run its fused
        # cascade (cascade_fwd_hl_f32 + the single-layer cached backward per block)
        hl = not any(flags) and F.cascade_hl_supported(n)
        return {"blocks": blocks, "flags": flags, "flags_t": torch.tensor(flags, dtype=torch.uint8, device=dev),
                "perm": perm, "perm_inv": perm_inv, "n": n, "device": dev, "hl": hl}

    @property
    def fused(self) -> bool:
        """True when forward/backward run the fused cascade kernels."""
        return self._fused is not None

    @property
    def n_in(self):
        return self.layers[0].n_in

    @property
    def n_out(self):
        return self.layers[-1].n_out

    def forward(self, x):
        host = not (isinstance(x, torch.Tensor) and x.is_cuda)
        if self._fused is not None:
            fz = self._fused
            xt, _ = self.layers[0]._check_input(x)
            acdc = [b[0] for b in fz["blocks"]]
            a = torch.stack([l.a for l in acdc])
            d = torch.stack([l.d for l in acdc])
            bias = torch.stack([l.bias_d for l in acdc])
            y, ckpt = F.cascade_forward(xt, a, d, bias, fz["perm"], fz["flags_t"], hl=fz["hl"])
            self._cache = (xt, ckpt)
            return Layer._out(y, host)
        if host:
            x, _ = self.layers[0]._check_input(x, torch.complex64 if self.complex_domain else torch.float32)
        for layer in self.layers:
            x = layer.forward(x)
        return Layer._out(x, host)

    def backward(self, grad_y, retain_cache=False, sgd=None, on_layer=None):
        """``sgd`` (fused stacks only, from ``training.Sgd.backward_step``): per
        block SGD specs; each block's optimizer step runs in its backward.
        ``on_layer(layer)`` is called once each layer's backward is enqueued
        (last layer first; in a fused stack for each ACDC layer of a block)."""
        host = not (isinstance(grad_y, torch.Tensor) and grad_y.is_cuda)
        if sgd is not None and self._fused is None:
            raise ValueError("a fused SGD backward needs a fused cascade")
        if self._fused is not None:
            if self._cache is None:
                raise RuntimeError("Cascade.backward called before forward")
            xt, ckpt = self._cache
            if not retain_cache:
                self._cache = None
            gy, _ = self.layers[-1]._check_input(grad_y)
            fz = self._fused
            acdc = [b[0] for b in fz["blocks"]]
            hook = (lambda l: on_layer(acdc[l])) if on_layer is not None else None
            dx = F.cascade_backward(xt, gy, [l.a for l in acdc], [l.d for l in acdc], fz["perm"], fz["flags"], ckpt,
                                    [(l.grad_a, l.grad_d, l.grad_bias_d) for l in acdc], accumulate=True, sgd=sgd,
                                    on_block=hook, perm_inv=fz["perm_inv"], hl=fz["hl"])
            return Layer._out(dx, host)
        g = grad_y
        if host:
            g, _ = self.layers[-1]._check_input(grad_y, torch.complex64 if self.complex_domain else torch.float32)
        for layer in reversed(self.layers):
            g = layer.backward(g, retain_cache=retain_cache)
            if on_layer is not None:
                on_layer(layer)
        return Layer._out(g, host)

    def params(self):
        out = []
        for layer in self.layers:
            out.extend(layer.params())
        return out

    def param_count(self):
        return sum(layer.param_count() for layer in self.layers)

    def zero_grads(self):
        for layer in self.layers:
            layer.zero_grads()


def acdc_cascade(n, depth, dct_mode="fast", backend="auto", device=None):
    """``depth`` identity-configured ACDC layers of size n (layers.py:360-362)."""
    return Cascade([AcdcLayer(n, dct_mode=dct_mode, backend=backend, device=device) for _ in range(depth)])


def afdf_cascade(n, depth, backend="auto", device=None):
    """``depth`` AFDF layers; the first signal diagonal is fixed (layers.py:365-370)."""
    return Cascade([AfdfLayer(n, backend=backend, fix_a=(i == 0), device=device) for i in range(depth)])


def count_params(obj):
    """3N per ACDC, 4N per AFDF, N*M+M per dense (layers.py:461-463)."""
    return obj.param_count()


# ------------------------------------------------------------ JSON interop
# The reference's on-disk cascade format (layers.py:466-554): one JSON document
# {"format_version": 1, "seed": ..., "layers": [spec, ...]} with float64 values.
# Parameters here are fp32: saving writes their exact values (so a file saved
# here reloads bit-exactly, here and in the reference); loading a reference
# file rounds each value to the nearest fp32.

def _tolist(t: torch.Tensor):
    return t.detach().to("cpu", dtype=torch.float64).tolist()


def _layer_spec(layer):
    if isinstance(layer, AcdcLayer):
        return {"type": "acdc", "n": layer.n_in, "dct_mode": layer.dct_mode, "a": _tolist(layer.a),
                "d": _tolist(layer.d), "bias_d": _tolist(layer.bias_d)}
    if isinstance(layer, AfdfLayer):
        return {"type": "afdf", "n": layer.n_in, "fix_a": layer.fix_a, "a_re": _tolist(layer.a.real),
                "a_im": _tolist(layer.a.imag), "d_re": _tolist(layer.d.real), "d_im": _tolist(layer.d.imag)}
    if isinstance(layer, ReluLayer):
        return {"type": "relu", "n": layer.n_in}
    if isinstance(layer, PermutationLayer):
        return {"type": "permutation", "n": layer.n_in, "perm": layer.perm.tolist()}
    if isinstance(layer, DenseLayer):
        return {"type": "dense", "n_in": layer.n_in, "n_out": layer.n_out, "w": _tolist(layer.w.reshape(-1)),
                "b": _tolist(layer.b)}
    raise TypeError(f"cannot serialize layer {type(layer).__name__}")


def _set(dst: torch.Tensor, values):
    dst.copy_(torch.as_tensor(np.asarray(values, dtype=np.float64).reshape(tuple(dst.shape))).to(dst.dtype))


def _layer_from_spec(spec, backend, device):
    tag = spec["type"]
    if tag == "acdc":
        layer = AcdcLayer(spec["n"], dct_mode=spec["dct_mode"], backend=backend, device=device)
        _set(layer.a, spec["a"])
        _set(layer.d, spec["d"])
        _set(layer.bias_d, spec["bias_d"])
        return layer
    if tag == "afdf":
        layer = AfdfLayer(spec["n"], backend=backend, fix_a=spec["fix_a"], device=device)
        a = np.asarray(spec["a_re"], dtype=np.float64) + 1j * np.asarray(spec["a_im"], dtype=np.float64)
        d = np.asarray(spec["d_re"], dtype=np.float64) + 1j * np.asarray(spec["d_im"], dtype=np.float64)
        layer.a.copy_(torch.as_tensor(a).to(torch.complex64))
        layer.d.copy_(torch.as_tensor(d).to(torch.complex64))
        return layer
    if tag == "relu":
        return ReluLayer(spec["n"], device=device)
    if tag == "permutation":
        return PermutationLayer(spec["n"], perm=spec["perm"], device=device)
    if tag == "dense":
        layer = DenseLayer(spec["n_in"], spec["n_out"], device=device)
        _set(layer.w, spec["w"])
        _set(layer.b, spec["b"])
        return layer
    raise ValueError(f"unknown layer tag {tag!r}")


def save_cascade(cascade, path, seed=None):
    """Write a cascade as the reference's JSON document (layers.py:536-545)."""
    doc = {"format_version": FORMAT_VERSION, "seed": seed, "layers": [_layer_spec(l) for l in cascade.layers]}
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(doc, fh)
        fh.write("\n")


def load_cascade(path, backend="auto", device=None):
    """Read a reference (or ``save_cascade``) JSON file into GPU layers (layers.py:548-554)."""
    with open(path, "r", encoding="utf-8") as fh:
        doc = json.load(fh)
    version = doc.get("format_version")
    if version != FORMAT_VERSION:
        raise ValueError(f"unsupported cascade format version {version!r}")
    return Cascade([_layer_from_spec(s, backend, device) for s in doc["layers"]])
