"""GPU tier: complex AFDF kernels vs the fp64 oracle and the reference's golden
vectors (layers.py:159-215).  Tolerances as for ACDC,
applied to complex magnitudes."""

import numpy as np
import pytest
import torch

from oracle import acdc_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda"


def c64(rng, *shape, mean=0.0, std=1.0):
    re = (mean + std * rng.standard_normal(shape)).astype(np.float32)
    im = (std * rng.standard_normal(shape)).astype(np.float32)
    return (re + 1j * im).astype(np.complex64)


def tc(a):
    return torch.as_tensor(np.asarray(a, dtype=np.complex64), device=DEV)


def check_rows(mine, ref, n, what):
    mine = mine.detach().cpu().numpy().astype(np.complex128)
    tol = O.fp32_tolerance(n, ref)
    err = float(np.abs(mine - ref).max())
    assert err <= tol, f"{what}: {err:.3e} > {tol:.3e} (N={n})"


def check_grad(mine, ref, n, rows, what):
    mine = mine.detach().cpu().numpy().astype(np.complex128)
    tol = O.grad_tolerance(n, rows, np.abs(ref))
    err = float(np.abs(mine - ref).max())
    assert err <= tol, f"{what}: {err:.3e} > {tol:.3e} (N={n}, B={rows})"


def run(x, dy, a, d, grads=None):
    from paper_1511_05946_b200 import functional as F

    n = a.shape[0]
    xt, dyt, at, dt = map(tc, (x, dy, a, d))
    y = F.afdf_forward(xt, at, dt)
    if grads is None:
        grads = [torch.zeros(n, dtype=torch.complex64, device=DEV) for _ in range(2)]
    dx = F.afdf_backward(xt, dyt, at, dt, *grads, accumulate=True)
    torch.cuda.synchronize()
    return y, dx, grads


@pytest.mark.parametrize("n,rows", [(2, 3), (4, 1), (8, 5), (16, 4), (32, 3), (64, 7), (128, 5), (256, 9),
                                    (1024, 33), (4096, 17), (8192, 12), (16384, 4)])
def test_afdf_vs_oracle(n, rows):
    rng = np.random.default_rng(77 + n)
    a, d = c64(rng, n, mean=1.0, std=0.3), c64(rng, n, mean=1.0, std=0.3)
    x, dy = c64(rng, rows, n), c64(rng, rows, n)
    y, dx, (ga, gd) = run(x, dy, a, d)
    X, A, D, DY = (v.astype(np.complex128) for v in (x, a, d, dy))
    yr, h2 = O.afdf_forward(X, A, D)
    dxr, gar, gdr = O.afdf_backward(X, h2, DY, A, D)
    check_rows(y, yr, n, "y")
    check_rows(dx, dxr, n, "dx")
    check_grad(ga, gar, n, rows, "grad_a")
    check_grad(gd, gdr, n, rows, "grad_d")


def test_afdf_golden(golden):
    cases = sorted({k[:-1] for k in golden.files if k.startswith("afdf_N") and k.endswith("_x")})
    assert cases
    for p in cases:
        g = lambda k: golden[p + k]
        n, rows = g("a").shape[0], g("x").shape[0]
        y, dx, (ga, gd) = run(g("x"), g("dy"), g("a"), g("d"))
        check_rows(y, g("y"), n, p + "y")
        check_rows(dx, g("dx"), n, p + "dx")
        check_grad(ga, g("ga"), n, rows, p + "ga")
        check_grad(gd, g("gd"), n, rows, p + "gd")


def test_afdf_layer_and_autograd():
    from paper_1511_05946_b200 import AfdfLayer, afdf, afdf_cascade

    n, rows = 256, 6
    rng = np.random.default_rng(3)
    layer = AfdfLayer(n, fix_a=True)
    assert len(layer.params()) == 1 and layer.param_count() == 4 * n
    x = c64(rng, rows, n)
    y = layer.forward(x)  # host in -> complex128 numpy out
    assert isinstance(y, np.ndarray) and y.dtype == np.complex128
    np.testing.assert_allclose(y, x.astype(np.complex128), atol=1e-5)  # identity init
    cas = afdf_cascade(n, 3)
    assert cas.complex_domain and cas.param_count() == 12 * n
    # autograd: torch complex autograd uses the same dL/dRe + i dL/dIm convention
    a = tc(c64(rng, n, mean=1.0, std=0.3)).requires_grad_()
    d = tc(c64(rng, n, mean=1.0, std=0.3)).requires_grad_()
    xt = tc(x).requires_grad_()
    w = tc(c64(rng, rows, n))
    out = afdf(xt, a, d)
    loss = (out * w.conj()).real.sum()
    loss.backward()
    X, A, D, W = (v.detach().cpu().numpy().astype(np.complex128) for v in (xt, a, d, w))
    yr, h2 = O.afdf_forward(X, A, D)
    dxr, gar, gdr = O.afdf_backward(X, h2, W, A, D)
    check_rows(xt.grad, dxr, n, "autograd dx")
    check_grad(a.grad, gar, n, rows, "autograd ga")
    check_grad(d.grad, gdr, n, rows, "autograd gd")
