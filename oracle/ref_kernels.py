"""Driver for the reference's own compiled CPU kernels (``oracle/_ref``).

TEST / BASELINE INFRASTRUCTURE.  Loads the Cython module built by
``oracle/build_ref.py`` (the reference's ``_kernels.pyx``, unmodified) and
drives it with the same call sequence as the reference layer code:

* ``RefAcdc.forward``  -> ``layers.py:141-146`` (dct2_batch, *d + b, dct3_batch)
* ``RefAcdc.backward`` -> ``layers.py:148-156``

Tables come from :class:`oracle.acdc_oracle.MakhoulTables`, the restatement of
``transforms.py:86-122`` (pinned against the reference by the golden tests).
Used for ``bench.py --impl reference`` (timed on the GPU box's host cores,
sharded over a thread pool: the Cython kernels release the GIL,
``_kernels.pyx:55,67,84``) and as a second oracle in the CPU tests.
"""

from __future__ import annotations

import glob
import importlib.machinery
import importlib.util
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from .acdc_oracle import tables

HERE = os.path.dirname(os.path.abspath(__file__))
_MOD = None


def load():
    """Return the compiled reference kernel module, or None if not built."""
    global _MOD
    if _MOD is not None:
        return _MOD
    hits = sorted(glob.glob(os.path.join(HERE, "_ref", "_kernels*.so")))
    if not hits:
        try:
            from .build_ref import build

            path = build()
        except Exception:  # pragma: no cover - build env missing
            path = None
        if not path or not os.path.exists(path):
            return None
        hits = [path]
    loader = importlib.machinery.ExtensionFileLoader("acdc._kernels", hits[0])
    spec = importlib.util.spec_from_file_location("acdc._kernels", hits[0], loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    _MOD = mod
    return mod


class RefAcdc:
    """One ACDC layer evaluated by the reference's compiled kernels (fp64)."""

    def __init__(self, a, d, bias):
        self.k = load()
        if self.k is None:
            raise RuntimeError("oracle/_ref is not built")
        self.a = np.ascontiguousarray(a, dtype=np.float64)
        self.d = np.ascontiguousarray(d, dtype=np.float64)
        self.bias = np.ascontiguousarray(bias, dtype=np.float64)
        self.t = tables(self.a.shape[0])

    def dct(self, x):
        out = np.empty_like(x)
        t = self.t
        self.k.dct2_batch(x, out, t.reorder, t.rev, t.tw, t.w4s)
        return out

    def idct(self, y):
        out = np.empty_like(y)
        t = self.t
        self.k.dct3_batch(y, out, t.reorder, t.rev, t.tw, t.u1, t.u2)
        return out

    def forward(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        h2 = self.dct(x * self.a)
        y = self.idct(h2 * self.d + self.bias)
        return y, h2

    def backward(self, x, h2, dy):
        dy = np.ascontiguousarray(dy, dtype=np.float64)
        g3 = self.dct(dy)
        gb = g3.sum(axis=0)
        gd = (h2 * g3).sum(axis=0)
        g1 = self.idct(g3 * self.d)
        ga = (x * g1).sum(axis=0)
        return g1 * self.a, ga, gd, gb


def fwd_bwd_threaded(layer: RefAcdc, x: np.ndarray, dy: np.ndarray, threads: int):
    """One forward+backward over ``x`` with rows sharded across ``threads``
    host threads; the per-shard parameter grads are summed in shard order
    (fixed-order reduction)."""
    rows = x.shape[0]
    bounds = np.linspace(0, rows, threads + 1).astype(int)

    def work(i):
        lo, hi = bounds[i], bounds[i + 1]
        if hi <= lo:
            return None
        xs = x[lo:hi]
        y, h2 = layer.forward(xs)
        dx, ga, gd, gb = layer.backward(xs, h2, dy[lo:hi])
        return y, dx, ga, gd, gb

    if threads == 1:
        parts = [work(0)]
    else:
        with ThreadPoolExecutor(threads) as ex:
            parts = list(ex.map(work, range(threads)))
    parts = [p for p in parts if p is not None]
    y = np.concatenate([p[0] for p in parts])
    dx = np.concatenate([p[1] for p in parts])
    ga = sum(p[2] for p in parts)
    gd = sum(p[3] for p in parts)
    gb = sum(p[4] for p in parts)
    return y, dx, ga, gd, gb


def ref_fft_rows(z: np.ndarray, inverse: bool, threads: int) -> np.ndarray:
    """Row-wise complex DFT by the reference's compiled ``fft_inplace``
    (``_kernels.pyx:49-57``; inverse scaled by 1/N, ``transforms.py:174-179``),
    rows sharded over ``threads`` host threads."""
    k = load()
    if k is None:
        raise RuntimeError("oracle/_ref is not built")
    z = np.array(z, dtype=np.complex128, order="C", copy=True)
    n = z.shape[1]
    t = tables(n)
    bounds = np.linspace(0, z.shape[0], threads + 1).astype(int)

    def work(i):
        lo, hi = bounds[i], bounds[i + 1]
        if hi > lo:
            k.fft_inplace(z[lo:hi], t.rev, t.tw, bool(inverse))

    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(work, range(threads)))
    return z


def afdf_fwd_bwd_threaded(x, dy, a, d, threads: int):
    """AFDF forward + backward (layers.py:199-215) with the reference's
    compiled FFT: returns y, dx, grad_a, grad_d (dL/dRe + i dL/dIm)."""
    n = x.shape[1]
    h2 = ref_fft_rows(x * a, False, threads)
    y = ref_fft_rows(h2 * d, True, threads)
    g3 = ref_fft_rows(dy, False, threads) / n
    gd = (g3 * np.conj(h2)).sum(axis=0)
    g1 = ref_fft_rows(g3 * np.conj(d), True, threads) * n
    ga = (g1 * np.conj(x)).sum(axis=0)
    return y, g1 * np.conj(a), ga, gd


def threads_available() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1
