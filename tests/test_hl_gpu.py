"""GPU tier: the half-length plan (hl_kernels.cu, N >= 1024:
one N/2-point complex FFT per row) against the fp64 oracle, with and without
the h2 cache, odd / single-row batches, the ACDC_HL=0 row-pair kernels as a
second implementation, and alignment handling at the C ABI.

Tolerances as tests/test_parity_gpu.py."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import acdc_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def f32(rng, *shape, mean=0.0, std=1.0):
    return (mean + std * rng.standard_normal(shape)).astype(np.float32)


@pytest.mark.parametrize("n,rows", [(n, r) for n in (1024, 2048, 4096, 8192, 16384, 32768) for r in (1, 4, 7)]
                         + [(1024, 601), (2048, 601), (4096, 601)])  # 601: many CTAs, leader reductions, idle groups
@pytest.mark.parametrize("cached", [True, False])
def test_hl_vs_oracle(n, rows, cached):
    from paper_1511_05946_b200 import functional as F

    rng = np.random.default_rng(n + rows)
    x, dy = f32(rng, rows, n), f32(rng, rows, n)
    a, d, b = f32(rng, n, mean=1.0, std=0.4), f32(rng, n, mean=1.0, std=0.4), f32(rng, n, std=0.3)
    t = lambda v: torch.as_tensor(v, device=DEV)
    hc = F.new_h2cache(rows, n, DEV) if cached else None
    y = F.acdc_forward(t(x), t(a), t(d), t(b), h2cache=hc)
    g = [torch.zeros(n, device=DEV) for _ in range(3)]
    dx = F.acdc_backward(t(x), t(dy), t(a), t(d), *g, accumulate=True, h2cache=hc)
    torch.cuda.synchronize()
    X, A, D, B, DY = (v.astype(np.float64) for v in (x, a, d, b, dy))
    yr, h2 = O.acdc_forward(X, A, D, B)
    dxr, gar, gdr, gbr = O.acdc_backward(X, h2, DY, A, D)
    for nm, m, r in (("y", y, yr), ("dx", dx, dxr)):
        e = float(np.abs(m.double().cpu().numpy() - r).max())
        assert e <= O.fp32_tolerance(n, r), f"{nm}: {e:.3e}"
    for nm, m, r in zip(("grad_a", "grad_d", "grad_bias"), g, (gar, gdr, gbr)):
        e = float(np.abs(m.double().cpu().numpy() - r).max())
        assert e <= O.grad_tolerance(n, rows, r), f"{nm}: {e:.3e}"


def test_hl_matches_row_pair_kernels():
    """Same inputs through ACDC_HL=0 (row-pair kernels) in a subprocess."""
    n, rows = 8192, 10
    rng = np.random.default_rng(3)
    arrs = [f32(rng, rows, n), f32(rng, rows, n), f32(rng, n, mean=1.0, std=0.3), f32(rng, n, mean=1.0, std=0.3),
            f32(rng, n, std=0.3)]
    path = os.path.join(ROOT, "gpurun_out", "hl_ab.npz") if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else \
        "/tmp/hl_ab.npz"
    np.savez(path, *arrs)
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {ROOT!r})
from paper_1511_05946_b200 import functional as F
z = np.load({path!r}); x, dy, a, d, b = (torch.as_tensor(z[f'arr_{{i}}'], device='cuda') for i in range(5))
y = F.acdc_forward(x, a, d, b)
g = [torch.zeros({n}, device='cuda') for _ in range(3)]
dx = F.acdc_backward(x, dy, a, d, *g)
np.savez({path!r} + '.out.npz', y=y.cpu().numpy(), dx=dx.cpu().numpy(), g=torch.stack(g).cpu().numpy())
"""
    res = {}
    for hl in ("1", "0"):
        env = dict(os.environ, ACDC_HL=hl)
        subprocess.run([sys.executable, "-c", code], env=env, check=True)
        res[hl] = dict(np.load(path + ".out.npz"))
    for k in ("y", "dx"):
        ref = res["0"][k].astype(np.float64)
        e = float(np.abs(res["1"][k] - ref).max())
        assert e <= 2 * O.fp32_tolerance(n, ref), (k, e)
    e = float(np.abs(res["1"]["g"] - res["0"]["g"]).max())
    assert e <= 2 * O.grad_tolerance(n, rows, res["0"]["g"].astype(np.float64)), e


def test_hl_alignment_at_the_abi():
    """Cached calls at an HL size with misaligned rows fail loudly
    (ACDC_E_ALIGN); uncached ones fall back to the row-pair kernels."""
    from paper_1511_05946_b200 import _lib
    from paper_1511_05946_b200 import functional as F

    n, rows = 8192, 3
    lib = _lib.load()
    buf = torch.randn(rows * (n + 2) + 2, device=DEV)
    x = buf[2:].as_strided((rows, n), (n + 2, 1))  # 8-byte aligned rows, ld % 4 == 2
    y = torch.empty(rows, n + 2, device=DEV)
    v = torch.ones(n, device=DEV)
    s = torch.cuda.current_stream().cuda_stream
    rc = lib.acdc_fwd_f32(x.data_ptr(), y.data_ptr(), v.data_ptr(), v.data_ptr(), torch.zeros(n, device=DEV).data_ptr(),
                          rows, n, n + 2, n + 2, s)
    assert rc == 0
    torch.cuda.synchronize()
    torch.testing.assert_close(y[:, :n], x, atol=1e-4, rtol=1e-4)  # identity layer
    hc = F.new_h2cache(rows, n, DEV)
    rc = lib.acdc_fwd_cache_f32(x.data_ptr(), y.data_ptr(), v.data_ptr(), v.data_ptr(),
                                torch.zeros(n, device=DEV).data_ptr(), hc.data_ptr(), rows, n, n + 2, n + 2, s)
    assert rc == _lib.ACDC_E_ALIGN
