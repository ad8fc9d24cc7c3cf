"""fp64 numpy restatement of the reference ACDC / AFDF hot path — TEST INFRASTRUCTURE.

This module is the parity oracle.  It re-derives, in plain numpy, the exact
algorithm the reference package runs on its compiled path, so that the CUDA
kernels can be checked against it on identical (fp32-representable) inputs.
It is imported only by ``tests/``, ``__graft_entry__.smoke()`` and the
CPU-baseline leg of ``bench.py``; the product path never calls it.

Parity is pinned (see ``tests/test_oracle.py``): this restatement is checked
against golden vectors produced by importing the reference itself
(``tests/golden/make_golden.py``) and against the SPEC known answers.

Reference map (paths relative to ``/root/reference/pkg/src/acdc``):

* ``bit_reversal``        -> ``transforms.py:43-49``
* ``dct_scales``          -> ``transforms.py:63-66``
* ``MakhoulTables``       -> ``transforms.py:86-122`` (fast-mode DctPlan tables)
* ``fft_rows``            -> ``_kernels.pyx:18-57`` / ``_kernels_py.py:17-40``
                             (radix-2 DIT, bit-reversed input, half-circle table)
* ``dct2_rows``           -> ``_kernels.pyx:60-73`` (reorder -> FFT -> Re(w4s * .))
* ``dct3_rows``           -> ``_kernels.pyx:76-91`` (pre-twiddle -> IFFT -> scatter)
* ``dct_matrix``          -> ``transforms.py:52-60`` (naive path, independent check)
* ``acdc_forward``        -> ``layers.py:141-146``
* ``acdc_backward``       -> ``layers.py:148-156`` (accumulating grads)
* ``afdf_forward/backward`` -> ``layers.py:199-215``
* ``relu_forward/backward`` -> ``layers.py:225-233`` (strict ``x > 0`` mask)
* ``perm_forward/backward`` -> ``layers.py:257-265`` (gather by perm / inverse)
* ``sgd_step``            -> ``training.py:72-84``
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "is_pow2",
    "bit_reversal",
    "dct_scales",
    "MakhoulTables",
    "fft_rows",
    "ifft_rows",
    "dct2_rows",
    "dct3_rows",
    "dct_matrix",
    "acdc_forward",
    "acdc_backward",
    "afdf_forward",
    "afdf_backward",
    "relu_forward",
    "relu_backward",
    "perm_forward",
    "perm_backward",
    "cascade_forward",
    "cascade_backward",
    "sgd_step",
    "fp32_tolerance",
    "grad_tolerance",
    "block_gain",
    "chain_factor",
]


def is_pow2(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


def bit_reversal(n: int) -> np.ndarray:
    """Bit-reversed index order (transforms.py:43-49), built by the same
    recurrence rev[i] = rev[i >> 1] >> 1 | (i & 1) << (bits - 1)."""
    bits = n.bit_length() - 1
    rev = np.zeros(n, dtype=np.int64)
    for i in range(1, n):
        rev[i] = (rev[i >> 1] >> 1) | ((i & 1) << max(bits - 1, 0))
    return rev


def dct_scales(n: int) -> np.ndarray:
    """Orthonormal scales s_0 = sqrt(1/N), s_k = sqrt(2/N) (transforms.py:63-66)."""
    s = np.full(n, math.sqrt(2.0 / n))
    s[0] = math.sqrt(1.0 / n)
    return s


class MakhoulTables:
    """Fast-mode DCT plan tables (transforms.py:86-122).

    * ``rev``     bit reversal for the size-N complex FFT
    * ``tw``      exp(-2 pi i k / N), k < max(N/2, 1)
    * ``reorder`` even indices ascending then odd indices descending
    * ``w4s``     s_k exp(-i pi k / 2N)        (DCT-II post-twiddle)
    * ``u1``      exp(+i pi k / 2N) / s_k      (DCT-III pre-twiddle, real part)
    * ``u2``      exp(+i pi k / 2N) sqrt(N/2), u2[0] = 0 (DCT-III mirror term)
    """

    def __init__(self, n: int):
        if not is_pow2(n):
            raise ValueError(f"fast DCT requires a power-of-two size, got {n}")
        self.n = n
        self.rev = bit_reversal(n)
        self.tw = np.exp(-2j * np.pi * np.arange(max(n // 2, 1)) / n)
        half = (n + 1) // 2
        order = np.empty(n, dtype=np.int64)
        order[:half] = np.arange(0, 2 * half, 2)
        order[half:] = 2 * (n - 1 - np.arange(half, n)) + 1
        self.reorder = order
        s = dct_scales(n)
        ph = np.pi * np.arange(n) / (2.0 * n)
        self.w4s = s * np.exp(-1j * ph)
        self.u1 = np.exp(1j * ph) / s
        u2 = np.exp(1j * ph) * math.sqrt(n / 2.0)
        u2[0] = 0.0
        self.u2 = u2


_TABLES: dict[int, MakhoulTables] = {}


def tables(n: int) -> MakhoulTables:
    t = _TABLES.get(n)
    if t is None:
        t = _TABLES[n] = MakhoulTables(n)
    return t


def _fft_core(z: np.ndarray, rev: np.ndarray, tw: np.ndarray, inverse: bool) -> np.ndarray:
    """Radix-2 decimation-in-time FFT over the last axis, vectorised over rows.

    Same numerics as ``_kernels.pyx:18-46``: bit-reversed input order,
    butterflies of span m = 2, 4, ..., N with twiddle tw[j * N/m]
    (conjugated for the inverse), inverse scaled by 1/N at the end.
    """
    b, n = z.shape
    out = z[:, rev].astype(np.complex128, copy=True)
    span = 2
    while span <= n:
        half = span // 2
        w = tw[0 : half * (n // span) : n // span]
        if inverse:
            w = np.conj(w)
        blk = out.reshape(b, n // span, span)
        lo = blk[:, :, :half].copy()
        hi = blk[:, :, half:] * w
        blk[:, :, :half] = lo + hi
        blk[:, :, half:] = lo - hi
        span *= 2
    if inverse:
        out *= 1.0 / n
    return out


def fft_rows(z: np.ndarray) -> np.ndarray:
    """Unnormalised forward DFT of each row (transforms.py:166-171)."""
    z = np.atleast_2d(np.asarray(z, dtype=np.complex128))
    t = _fft_tables(z.shape[1])
    return _fft_core(z, t[0], t[1], False)


def ifft_rows(z: np.ndarray) -> np.ndarray:
    """Inverse DFT of each row scaled by 1/N (transforms.py:174-179)."""
    z = np.atleast_2d(np.asarray(z, dtype=np.complex128))
    t = _fft_tables(z.shape[1])
    return _fft_core(z, t[0], t[1], True)


_FFT_T: dict[int, tuple] = {}


def _fft_tables(n: int):
    if not is_pow2(n):
        raise ValueError(f"FFT size must be a power of two, got {n}")
    t = _FFT_T.get(n)
    if t is None:
        t = _FFT_T[n] = (bit_reversal(n), np.exp(-2j * np.pi * np.arange(max(n // 2, 1)) / n))
    return t


def dct2_rows(x: np.ndarray) -> np.ndarray:
    """Orthonormal DCT-II of each row via Makhoul (``_kernels.pyx:60-73``)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    t = tables(x.shape[1])
    v = _fft_core(x[:, t.reorder].astype(np.complex128), t.rev, t.tw, False)
    return (v * t.w4s).real.copy()


def dct3_rows(y: np.ndarray) -> np.ndarray:
    """Orthonormal DCT-III (inverse of dct2_rows) (``_kernels.pyx:76-91``)."""
    y = np.atleast_2d(np.asarray(y, dtype=np.float64))
    n = y.shape[1]
    t = tables(n)
    v = np.empty(y.shape, dtype=np.complex128)
    v[:, 0] = t.u1[0] * y[:, 0]
    if n > 1:
        v[:, 1:] = t.u1[1:] * y[:, 1:] - 1j * (t.u2[1:] * y[:, :0:-1])
    v = _fft_core(v, t.rev, t.tw, True)
    out = np.empty_like(y)
    out[:, t.reorder] = v.real
    return out


def dct_matrix(n: int) -> np.ndarray:
    """Explicit orthonormal DCT-II matrix (transforms.py:52-60), rows n, cols k."""
    k = np.arange(n)
    c = math.sqrt(2.0 / n) * np.cos(np.pi * (2 * k[:, None] + 1) * k[None, :] / (2.0 * n))
    c[:, 0] /= math.sqrt(2.0)
    return c


# ---------------------------------------------------------------- layers


def acdc_forward(x, a, d, bias):
    """y = C3(d * C2(a * x) + bias); returns (y, h2) (layers.py:141-146)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    h2 = dct2_rows(x * a)
    y = dct3_rows(h2 * d + bias)
    return y, h2


def acdc_backward(x, h2, dy, a, d, grads=None):
    """Backward of acdc_forward (layers.py:148-156).

    Returns (dx, grad_a, grad_d, grad_bias).  If ``grads`` is a tuple of three
    arrays, the parameter gradients are accumulated into it (``+=``), matching
    the reference's accumulate-never-overwrite contract.
    """
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    dy = np.atleast_2d(np.asarray(dy, dtype=np.float64))
    g3 = dct2_rows(dy)
    gb = g3.sum(axis=0)
    gd = (h2 * g3).sum(axis=0)
    g1 = dct3_rows(g3 * d)
    ga = (x * g1).sum(axis=0)
    if grads is not None:
        grads[0][...] += ga
        grads[1][...] += gd
        grads[2][...] += gb
    return g1 * a, ga, gd, gb


def afdf_forward(x, a, d):
    """y = IFFT(d * FFT(a * x)); returns (y, h2) (layers.py:199-204)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.complex128))
    h2 = fft_rows(x * a)
    return ifft_rows(h2 * d), h2


def afdf_backward(x, h2, dy, a, d):
    """Backward of afdf_forward with the conj-adjoint convention
    dL/dRe + i dL/dIm (layers.py:206-215).  Returns (dx, grad_a, grad_d)."""
    x = np.atleast_2d(np.asarray(x, dtype=np.complex128))
    dy = np.atleast_2d(np.asarray(dy, dtype=np.complex128))
    n = x.shape[1]
    g3 = fft_rows(dy) / n
    gd = (g3 * np.conj(h2)).sum(axis=0)
    g1 = ifft_rows(g3 * np.conj(d)) * n
    ga = (g1 * np.conj(x)).sum(axis=0)
    return g1 * np.conj(a), ga, gd


def relu_forward(x):
    """max(x, 0) with the strict x > 0 mask (layers.py:225-228)."""
    x = np.asarray(x, dtype=np.float64)
    return np.maximum(x, 0.0), x > 0


def relu_backward(dy, mask):
    return np.asarray(dy, dtype=np.float64) * mask


def perm_forward(x, perm):
    """y[:, j] = x[:, perm[j]] (layers.py:257-261)."""
    return np.ascontiguousarray(np.asarray(x)[:, perm])


def perm_backward(dy, perm):
    """dx = dy[:, argsort(perm)] (layers.py:254, 263-265)."""
    return np.ascontiguousarray(np.asarray(dy)[:, np.argsort(perm)])


def cascade_forward(x, layers):
    """Run a list of layer specs in order (layers.py:336-339).

    Each spec is a dict: {"kind": "acdc", "a", "d", "bias"} | {"kind": "relu"}
    | {"kind": "perm", "perm"}.  Returns (y, caches)."""
    caches = []
    for spec in layers:
        kind = spec["kind"]
        if kind == "acdc":
            y, h2 = acdc_forward(x, spec["a"], spec["d"], spec["bias"])
            caches.append((x, h2))
        elif kind == "relu":
            y, mask = relu_forward(x)
            caches.append(mask)
        elif kind == "perm":
            y = perm_forward(x, spec["perm"])
            caches.append(None)
        else:
            raise ValueError(kind)
        x = y
    return x, caches


def cascade_backward(dy, layers, caches):
    """Reverse pass (layers.py:341-344).  Returns (dx, per-layer grads)."""
    grads = [None] * len(layers)
    for i in range(len(layers) - 1, -1, -1):
        spec, cache = layers[i], caches[i]
        kind = spec["kind"]
        if kind == "acdc":
            x, h2 = cache
            dy, ga, gd, gb = acdc_backward(x, h2, dy, spec["a"], spec["d"])
            grads[i] = (ga, gd, gb)
        elif kind == "relu":
            dy = relu_backward(dy, cache)
        else:
            dy = perm_backward(dy, spec["perm"])
    return dy, grads


def sgd_step(value, grad, velocity, lr, momentum=0.0, weight_decay=0.0, decay=False, lr_mult=1.0):
    """Momentum SGD (training.py:72-84): v = mu v - lr*lr_mult*(g + wd p [decay]);
    p += v; grad = 0.  Operates in place on numpy arrays."""
    g = grad + weight_decay * value if (weight_decay != 0.0 and decay) else grad
    velocity *= momentum
    velocity -= (lr * lr_mult) * g
    value += velocity
    grad[...] = 0


# ------------------------------------------------------------- tolerances

EPS32 = 2.0**-23


def fp32_tolerance(n: int, ref: np.ndarray) -> float:
    """Max-abs bound for fp32 y / dx against the fp64 oracle:
    4 * log2(N) * eps32 * max(rms(ref), 1)."""
    lg = max(1.0, math.log2(max(n, 2)))
    rms = float(np.sqrt(np.mean(np.abs(ref) ** 2))) if ref.size else 0.0
    return 4.0 * lg * EPS32 * max(rms, 1.0)


def grad_tolerance(n: int, rows: int, ref: np.ndarray) -> float:
    """Max-abs bound for batch-reduced parameter grads:
    4 * (log2 N + log2 B) * eps32 * max(|ref|_inf, 1) ... with a floor of one
    ulp-scale term for tiny references."""
    lg = max(1.0, math.log2(max(n, 2))) + max(1.0, math.log2(max(rows, 2)))
    mx = float(np.max(np.abs(ref))) if ref.size else 0.0
    return 4.0 * lg * EPS32 * max(mx, 1.0)


def block_gain(a, d) -> float:
    """rms gain of one ACDC block on an error vector e (layers.py:141-146):
    C is orthonormal, so ||C3(d * C2(a * e))||_2 = ||d * C2(a * e)||_2, which
    for rounding errors uncorrelated with the diagonals is rms(a) * rms(d) *
    ||e||_2.  ReLU (1-Lipschitz) and permutations (isometries) add no gain."""
    a, d = np.asarray(a), np.asarray(d)
    return float(np.sqrt(np.mean(np.abs(a) ** 2) * np.mean(np.abs(d) ** 2)))


def chain_factor(gains) -> float:
    """Error bound multiplier for a chain of K blocks, each adding at most the
    single-layer rounding bound and passing the incoming error on through its
    gain: sum_{l<K} prod_{l<k<K} g_k (gains in propagation order).  For a
    cascade's y this is applied to fp32_tolerance (the per-block bound); for dx
    with the backward's order of gains."""
    total, prod = 0.0, 1.0
    for g in reversed(list(gains)):
        total += prod
        prod *= g
    return total
