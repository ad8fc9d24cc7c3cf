"""Transform plans with the reference's attributes (transforms.py:69-122) and
the kernel-backend selection of backend.py:30-42.

``DctPlan`` / ``FftPlan`` keep the host tables the reference plans expose
(``bitrev``, ``twiddle``, ``reorder``, ``w4s``, ``u1``, ``u2``; ``cos_matrix``
in naive mode), so code that inspects a layer's plan keeps working.  The
B200 kernels build their own fp32 device tables from the same formulas
(csrc/runtime.cu, computed in fp64 and rounded once); these host copies are
what the plan reports, not what the kernels read.

Backends: the reference accepts "auto" | "compiled" | "python" (and the env
override ``ACDC_KERNEL_BACKEND``); every one of them selects the same
numerics, so here all of them, plus "b200", resolve to the sm_100a kernels
(``plan.backend == "b200"``).  An unknown name raises the reference's
ValueError.  There is no CPU fallback.
"""

from __future__ import annotations

import os

import numpy as np
import torch

BACKENDS = ("auto", "compiled", "python", "b200")


def resolve_backend(name: str = "auto") -> str:
    """backend.py:30-42 semantics: "auto" honours ACDC_KERNEL_BACKEND."""
    if name == "auto":
        name = os.environ.get("ACDC_KERNEL_BACKEND", "auto")
    if name not in BACKENDS:
        raise ValueError(f"unknown kernel backend {name!r}, expected one of {BACKENDS}")
    return "b200"


def is_power_of_two(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


def bit_reversal_permutation(n: int) -> np.ndarray:
    """Bit-reversed index order for a power-of-two n (transforms.py:43-49)."""
    bits = max(int(n).bit_length() - 1, 0)
    rev = np.zeros(n, dtype=np.int64)
    for i in range(1, n):
        rev[i] = (rev[i >> 1] >> 1) | ((i & 1) << (bits - 1))
    return rev


def dct_matrix(n: int) -> np.ndarray:
    """Orthonormal DCT-II matrix, rows indexed by n, columns by k (transforms.py:52-60)."""
    if n <= 0:
        raise ValueError(f"size must be positive, got {n}")
    kk = np.arange(n)
    c = np.sqrt(2.0 / n) * np.cos(np.pi * (2 * kk[:, None] + 1) * kk / (2.0 * n))
    c[:, 0] /= np.sqrt(2.0)
    return c


class FftPlan:
    """Bit reversal and half-circle twiddles for a power-of-two size (transforms.py:69-83)."""

    def __init__(self, n, backend="auto"):
        if not is_power_of_two(n):
            raise ValueError(f"FFT size must be a power of two, got {n}")
        self.n = n
        self.backend = resolve_backend(backend)
        self.bitrev = bit_reversal_permutation(n)
        self.twiddle = np.exp(-2j * np.pi * np.arange(max(n // 2, 1)) / n)


class DctPlan:
    """DCT plan in ``naive`` (cosine matrix) or ``fast`` (Makhoul FFT) mode
    (transforms.py:86-122)."""

    MODES = ("naive", "fast")

    def __init__(self, n, mode="fast", backend="auto"):
        if n <= 0:
            raise ValueError(f"size must be positive, got {n}")
        if mode not in self.MODES:
            raise ValueError(f"unknown DCT mode {mode!r}, expected one of {self.MODES}")
        if mode == "fast" and not is_power_of_two(n):
            raise ValueError(f"fast DCT requires a power-of-two size, got {n}")
        self.n = n
        self.mode = mode
        self._dev_cos = {}
        if mode == "naive":
            self.cos_matrix = dct_matrix(n)
            self.backend = "naive"
            return
        self.backend = resolve_backend(backend)
        self.bitrev = bit_reversal_permutation(n)
        self.twiddle = np.exp(-2j * np.pi * np.arange(max(n // 2, 1)) / n)
        reorder = np.empty(n, dtype=np.int64)
        top = (n + 1) // 2
        reorder[:top] = 2 * np.arange(top)
        reorder[top:] = 2 * (n - 1 - np.arange(top, n)) + 1
        self.reorder = reorder
        s = np.full(n, np.sqrt(2.0 / n))
        s[0] = np.sqrt(1.0 / n)
        phase = np.pi * np.arange(n) / (2.0 * n)
        self.w4s = s * np.exp(-1j * phase)
        self.u1 = np.exp(1j * phase) / s
        u2 = np.zeros(n, dtype=np.complex128)
        if n > 1:
            u2[1:] = np.exp(1j * phase[1:]) * np.sqrt(n / 2.0)
        self.u2 = u2

    def cos_device(self, device) -> torch.Tensor:
        """fp32 copy of the cosine matrix on ``device`` (naive mode; built once)."""
        key = str(device)
        c = self._dev_cos.get(key)
        if c is None:
            c = self._dev_cos[key] = torch.as_tensor(self.cos_matrix, dtype=torch.float32, device=device)
        return c
