"""GPU tier: the sm_100a kernels through the C ABI vs the fp64 oracle.

Tolerances: y, dx max-abs <= 4*log2(N)*eps32*max(rms(ref),1);
parameter grads max-abs <= 4*(log2 N + log2 B)*eps32*max(|ref|_inf, 1).
Inputs are fp32; the oracle runs on the same values up-cast to fp64.
"""

import numpy as np
import pytest
import torch

from oracle import acdc_oracle as O

pytestmark = pytest.mark.gpu

DEV = "cuda"


def t32(a):
    return torch.as_tensor(np.asarray(a, dtype=np.float32), device=DEV)


def f32(rng, *shape, mean=0.0, std=1.0):
    return (mean + std * rng.standard_normal(shape)).astype(np.float32)


def assert_close_rows(mine, ref, n, what):
    mine = mine.detach().cpu().double().numpy() if isinstance(mine, torch.Tensor) else mine
    tol = O.fp32_tolerance(n, ref)
    err = float(np.abs(mine - ref).max()) if ref.size else 0.0
    assert err <= tol, f"{what}: max err {err:.3e} > tol {tol:.3e} (N={n})"


def assert_close_grad(mine, ref, n, rows, what):
    mine = mine.detach().cpu().double().numpy()
    tol = O.grad_tolerance(n, rows, ref)
    err = float(np.abs(mine - ref).max())
    assert err <= tol, f"{what}: max err {err:.3e} > tol {tol:.3e} (N={n}, B={rows})"


def run_acdc(x, dy, a, d, b, accumulate_into=None):
    from paper_1511_05946_b200 import functional as F

    n = a.shape[0]
    xt, dyt, at, dt, bt = map(t32, (x, dy, a, d, b))
    y = F.acdc_forward(xt, at, dt, bt)
    if accumulate_into is None:
        grads = [torch.zeros(n, device=DEV) for _ in range(3)]
    else:
        grads = accumulate_into
    dx = F.acdc_backward(xt, dyt, at, dt, *grads, accumulate=True)
    torch.cuda.synchronize()
    return y, dx, grads


@pytest.mark.parametrize("n", [2 ** k for k in range(1, 16)])
def test_dct_idct_sweep(n):
    from paper_1511_05946_b200 import functional as F

    rng = np.random.default_rng(n)
    rows = 5 if n <= 4096 else 3
    x = f32(rng, rows, n)
    ref2, ref3 = O.dct2_rows(x.astype(np.float64)), O.dct3_rows(x.astype(np.float64))
    assert_close_rows(F.dct(t32(x)), ref2, n, "dct")
    assert_close_rows(F.idct(t32(x)), ref3, n, "idct")


@pytest.mark.parametrize("n,rows", [(1, 7), (2, 1), (4, 3), (8, 2), (16, 5), (32, 4), (64, 9), (128, 16), (256, 128),
                                    (512, 33), (1024, 64), (2048, 17), (4096, 64), (8192, 12), (16384, 6),
                                    (32768, 3)])
def test_acdc_fwd_bwd_vs_oracle(n, rows):
    rng = np.random.default_rng(1000 + n)
    a, d = f32(rng, n, mean=1.0, std=0.4), f32(rng, n, mean=1.0, std=0.4)
    b = f32(rng, n, std=0.3)
    x, dy = f32(rng, rows, n), f32(rng, rows, n)
    y, dx, (ga, gd, gb) = run_acdc(x, dy, a, d, b)
    X, A, D, Bb, DY = (v.astype(np.float64) for v in (x, a, d, b, dy))
    yr, h2 = O.acdc_forward(X, A, D, Bb)
    dxr, gar, gdr, gbr = O.acdc_backward(X, h2, DY, A, D)
    assert_close_rows(y, yr, n, "y")
    assert_close_rows(dx, dxr, n, "dx")
    assert_close_grad(ga, gar, n, rows, "grad_a")
    assert_close_grad(gd, gdr, n, rows, "grad_d")
    assert_close_grad(gb, gbr, n, rows, "grad_bias")


def test_golden_acdc(golden):
    cases = sorted({k[:-1] for k in golden.files if k.startswith("acdc_N") and k.endswith("_x")})
    for p in cases:
        g = lambda k: golden[p + k]
        n, rows = g("a").shape[0], g("x").shape[0]
        grads = [torch.zeros(n, device=DEV) for _ in range(3)]
        y, dx, _ = run_acdc(g("x"), g("dy"), g("a"), g("d"), g("bias"), grads)
        assert_close_rows(y, g("y"), n, p + "y")
        assert_close_rows(dx, g("dx"), n, p + "dx")
        assert_close_grad(grads[0], g("ga"), n, rows, p + "ga")
        assert_close_grad(grads[1], g("gd"), n, rows, p + "gd")
        assert_close_grad(grads[2], g("gb"), n, rows, p + "gb")
        # second backward accumulates (layers.py:152-155)
        run_acdc(g("x"), g("dy"), g("a"), g("d"), g("bias"), grads)
        assert_close_grad(grads[0], g("ga2"), n, rows, p + "ga2")
        assert_close_grad(grads[1], g("gd2"), n, rows, p + "gd2")
        assert_close_grad(grads[2], g("gb2"), n, rows, p + "gb2")


def test_golden_dct(golden):
    from paper_1511_05946_b200 import functional as F

    for k in golden.files:
        if k.startswith("dct_N") and k.endswith("_x"):
            p = k[:-1]
            n = golden[k].shape[1]
            assert_close_rows(F.dct(t32(golden[k])), golden[p + "dct"], n, p)
            assert_close_rows(F.idct(t32(golden[k])), golden[p + "idct"], n, p)


def test_known_answers():
    from paper_1511_05946_b200 import functional as F

    n = 4096
    ones = torch.ones(3, n, device=DEV)
    out = F.dct(ones).cpu().double().numpy()
    assert abs(out[0, 0] - 64.0) < 1e-4 and np.abs(out[:, 1:]).max() < 1e-4
    rng = np.random.default_rng(5)
    x = f32(rng, 8, n)
    one, zero = np.ones(n, np.float32), np.zeros(n, np.float32)
    y, dx, grads = run_acdc(x, x, one, one, zero)
    assert_close_rows(y, x.astype(np.float64), n, "identity y")
    assert_close_rows(dx, x.astype(np.float64), n, "identity dx")
    bias = f32(rng, n)
    y0, _, _ = run_acdc(x, x, zero, one, bias)
    ref = O.dct3_rows(bias.astype(np.float64)[None])[0]
    assert_close_rows(y0, np.broadcast_to(ref, (8, n)), n, "a=0")
    _, dx0, (ga, gd, gb) = run_acdc(x, np.zeros_like(x), one, one, zero)
    assert float(dx0.abs().max()) == 0 and float(ga.abs().max()) == 0
    assert float(gd.abs().max()) == 0 and float(gb.abs().max()) == 0


def test_grads_deterministic_and_accumulate():
    rng = np.random.default_rng(9)
    n, rows = 4096, 2048 + 1  # odd row count exercises the half-empty row pair
    a, d, b = f32(rng, n, mean=1, std=0.1), f32(rng, n, mean=1, std=0.1), f32(rng, n, std=0.1)
    x, dy = f32(rng, rows, n), f32(rng, rows, n)
    _, dx1, g1 = run_acdc(x, dy, a, d, b)
    _, dx2, g2 = run_acdc(x, dy, a, d, b)
    assert torch.equal(dx1, dx2)
    for u, v in zip(g1, g2):
        assert torch.equal(u, v), "gradients must be bitwise deterministic"
    g_acc = [g.clone() for g in g1]
    run_acdc(x, dy, a, d, b, g_acc)
    for u, v in zip(g_acc, g1):
        torch.testing.assert_close(u, 2 * v, rtol=1e-6, atol=1e-5)


def test_strided_rows_and_errors():
    from paper_1511_05946_b200 import functional as F

    n = 256
    rng = np.random.default_rng(3)
    big = t32(f32(rng, 6, 2 * n))
    view = big[:, :n]  # ld = 2n
    assert view.stride(0) == 2 * n
    a, d, b = (torch.ones(n, device=DEV) for _ in range(3))
    b.zero_()
    y = F.acdc_forward(view, a, d, b)
    assert_close_rows(y, view.cpu().double().numpy(), n, "strided identity")
    with pytest.raises(ValueError):
        F.acdc_forward(torch.ones(4, 12, device=DEV), *(torch.ones(12, device=DEV) for _ in range(3)))


def test_layer_api_matches_reference_contract(golden):
    from paper_1511_05946_b200 import AcdcLayer

    p = "acdc_N256_B4_"
    g = lambda k: golden[p + k]
    layer = AcdcLayer(256)
    layer.a.copy_(t32(g("a")))
    layer.d.copy_(t32(g("d")))
    layer.bias_d.copy_(t32(g("bias")))
    with pytest.raises(RuntimeError, match="backward called before forward"):
        layer.backward(g("dy"))
    y = layer.forward(g("x"))  # host numpy in -> numpy float64 out
    assert isinstance(y, np.ndarray) and y.dtype == np.float64
    assert_close_rows(y, g("y"), 256, "layer y")
    dx = layer.backward(g("dy"), retain_cache=True)
    assert_close_rows(dx, g("dx"), 256, "layer dx")
    layer.backward(g("dy"))
    assert_close_grad(layer.grad_a, g("ga2"), 256, 4, "layer ga2")
    with pytest.raises(RuntimeError):
        layer.backward(g("dy"))
    layer.zero_grads()
    assert float(layer.grad_a.abs().sum()) == 0
    with pytest.raises(ValueError, match="expects"):
        layer.forward(np.ones((2, 128)))
    with pytest.raises(ValueError, match="power-of-two"):
        AcdcLayer(100)


@pytest.mark.parametrize("n,rows", [(128, 9), (512, 37), (4096, 64)])  # recompute / h2 cache / TMEM backward
def test_autograd_function(n, rows):
    from paper_1511_05946_b200 import acdc

    rng = np.random.default_rng(11)
    x = t32(f32(rng, rows, n)).requires_grad_()
    a = t32(f32(rng, n, mean=1, std=0.3)).requires_grad_()
    d = t32(f32(rng, n, mean=1, std=0.3)).requires_grad_()
    b = t32(f32(rng, n, std=0.3)).requires_grad_()
    y = acdc(x, a, d, b)
    w = t32(f32(rng, rows, n))
    (y * w).sum().backward()
    X, A, D, B, W = (v.detach().cpu().double().numpy() for v in (x, a, d, b, w))
    yr, h2 = O.acdc_forward(X, A, D, B)
    dxr, gar, gdr, gbr = O.acdc_backward(X, h2, W, A, D)
    assert_close_rows(y, yr, n, "autograd y")
    assert_close_rows(x.grad, dxr, n, "autograd dx")
    assert_close_grad(a.grad, gar, n, rows, "autograd ga")
    assert_close_grad(d.grad, gdr, n, rows, "autograd gd")
    assert_close_grad(b.grad, gbr, n, rows, "autograd gb")


@pytest.mark.parametrize("n,rows", [(256, 7), (1024, 64), (4096, 33), (8192, 5), (16384, 3)])
def test_h2cache_matches_recompute(n, rows):
    """h2-cache forward/backward (layers.py:145 cache semantics) == recompute path."""
    from paper_1511_05946_b200 import functional as F

    rng = np.random.default_rng(2000 + n)
    a, d, b = f32(rng, n, mean=1, std=0.4), f32(rng, n, mean=1, std=0.4), f32(rng, n, std=0.3)
    x, dy = f32(rng, rows, n), f32(rng, rows, n)
    xt, dyt, at, dt, bt = map(t32, (x, dy, a, d, b))
    cache = F.new_h2cache(rows, n, DEV)
    y = F.acdc_forward(xt, at, dt, bt, h2cache=cache)
    g = [torch.zeros(n, device=DEV) for _ in range(3)]
    dx = F.acdc_backward(xt, dyt, at, dt, *g, h2cache=cache)
    torch.cuda.synchronize()
    X, A, D, B, DY = (v.astype(np.float64) for v in (x, a, d, b, dy))
    yr, h2 = O.acdc_forward(X, A, D, B)
    dxr, gar, gdr, gbr = O.acdc_backward(X, h2, DY, A, D)
    assert_close_rows(y, yr, n, "y")
    assert_close_rows(dx, dxr, n, "dx")
    assert_close_grad(g[0], gar, n, rows, "grad_a")
    assert_close_grad(g[1], gdr, n, rows, "grad_d")
    assert_close_grad(g[2], gbr, n, rows, "grad_bias")
    with pytest.raises(ValueError):
        F.new_h2cache(4, 128, DEV)


@pytest.mark.parametrize("chunks,nbuf,ramp,direct", [(5, 2, False, False), (16, 3, True, False), (7, 2, False, True)])
def test_host_pipeline_matches_device_path(chunks, nbuf, ramp, direct):
    """functional.HostPipeline (chunked H2D / kernels / D2H overlap, or kernels
    storing straight into mapped host memory) == one device call."""
    from paper_1511_05946_b200 import functional as F

    n, rows = 1024, 300
    rng = np.random.default_rng(21)
    x, dy = f32(rng, rows, n), f32(rng, rows, n)
    a, d, b = (t32(f32(rng, n, mean=m, std=0.3)) for m in (1.0, 1.0, 0.0))
    pipe = F.HostPipeline(n, rows, DEV, chunks=chunks, nbuf=nbuf, ramp=ramp, direct_out=direct)
    assert sum(hi - lo for lo, hi in pipe.spans) == rows
    xh, dyh = torch.as_tensor(x).pin_memory(), torch.as_tensor(dy).pin_memory()
    yh, dxh = torch.empty(rows, n).pin_memory(), torch.empty(rows, n).pin_memory()
    g = [torch.zeros(n, device=DEV) for _ in range(3)]
    pipe.step(xh, dyh, yh, dxh, a, d, b, g, accumulate=False)
    torch.cuda.synchronize()
    g2 = [torch.zeros(n, device=DEV) for _ in range(3)]
    y2 = F.acdc_forward(t32(x), a, d, b)
    dx2 = F.acdc_backward(t32(x), t32(dy), a, d, *g2)
    torch.cuda.synchronize()
    # chunks start on even rows (same row pairing as one call): bit-identical
    torch.testing.assert_close(yh, y2.cpu(), rtol=0, atol=0)
    torch.testing.assert_close(dxh, dx2.cpu(), rtol=0, atol=0)
    for u, v in zip(g, g2):
        torch.testing.assert_close(u, v, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("overlap", [True, False])
def test_host_pipeline_consecutive_steps(overlap):
    """Back-to-back HostPipeline steps with different inputs and outputs: with
    overlap_steps a step's uploads run under the previous step's downloads, so
    every step's y, dx and gradients must still equal its own device call."""
    from paper_1511_05946_b200 import functional as F

    n, rows, steps = 2048, 1000, 3
    rng = np.random.default_rng(33)
    a, d, b = (t32(f32(rng, n, mean=m, std=0.3)) for m in (1.0, 1.0, 0.0))
    pipe = F.HostPipeline(n, rows, DEV, chunks=4, overlap_steps=overlap)
    xs = [torch.as_tensor(f32(rng, rows, n)).pin_memory() for _ in range(steps)]
    dys = [torch.as_tensor(f32(rng, rows, n)).pin_memory() for _ in range(steps)]
    ys = [torch.empty(rows, n).pin_memory() for _ in range(steps)]
    dxs = [torch.empty(rows, n).pin_memory() for _ in range(steps)]
    gs = [[torch.zeros(n, device=DEV) for _ in range(3)] for _ in range(steps)]
    for i in range(steps):  # no host sync between steps
        pipe.step(xs[i], dys[i], ys[i], dxs[i], a, d, b, gs[i], accumulate=False)
    torch.cuda.synchronize()
    for i in range(steps):
        g2 = [torch.zeros(n, device=DEV) for _ in range(3)]
        y2 = F.acdc_forward(xs[i].to(DEV), a, d, b)
        dx2 = F.acdc_backward(xs[i].to(DEV), dys[i].to(DEV), a, d, *g2)
        torch.cuda.synchronize()
        torch.testing.assert_close(ys[i], y2.cpu(), rtol=0, atol=0)
        torch.testing.assert_close(dxs[i], dx2.cpu(), rtol=0, atol=0)
        for u, v in zip(gs[i], g2):
            torch.testing.assert_close(u, v, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("n,rows", [(1024, 4096), (4096, 2048)])
def test_backward_of_forward_output_back_to_back(n, rows):
    """backward(dy = y) launched right after the forward that writes y: the
    backward starts early under programmatic dependent launch and must not read
    y (or the h2 cache) before the forward has finished."""
    from paper_1511_05946_b200 import functional as F

    rng = np.random.default_rng(n)
    x = f32(rng, rows, n)
    a, d, b = f32(rng, n, mean=1.0, std=0.2), f32(rng, n, mean=1.0, std=0.2), f32(rng, n, std=0.2)
    xt, at, dt, bt = t32(x), t32(a), t32(d), t32(b)
    hc = F.new_h2cache(rows, n, DEV)
    g = [torch.zeros(n, device=DEV) for _ in range(3)]
    for _ in range(3):  # repeated: the race, if any, would show on some launch
        y = F.acdc_forward(xt, at, dt, bt, h2cache=hc)
        dx = F.acdc_backward(xt, y, at, dt, *g, accumulate=False, h2cache=hc)
    torch.cuda.synchronize()
    X, A, D, B = (v.astype(np.float64) for v in (x, a, d, b))
    yr, h2 = O.acdc_forward(X, A, D, B)
    dxr, gar, gdr, gbr = O.acdc_backward(X, h2, y.double().cpu().numpy(), A, D)
    assert_close_rows(y, yr, n, "y")
    assert_close_rows(dx, dxr, n, "dx")
    for mine, ref, nm in zip(g, (gar, gdr, gbr), ("grad_a", "grad_d", "grad_bias")):
        assert_close_grad(mine, ref, n, rows, nm)


@pytest.mark.parametrize("pad", [2, 4])
def test_cached_backward_strided_dy(pad):
    """Cached backward with dy rows at a leading dimension n + pad: pad = 4 keeps
    16-byte row alignment (dy is bulk-copied into shared memory), pad = 2 does
    not (dy is loaded directly)."""
    from paper_1511_05946_b200 import functional as F

    n, rows = 1024, 37
    rng = np.random.default_rng(pad)
    x, dy = f32(rng, rows, n), f32(rng, rows, n)
    a, d, b = f32(rng, n, mean=1.0, std=0.2), f32(rng, n, mean=1.0, std=0.2), f32(rng, n, std=0.2)
    wide = torch.zeros(rows, n + pad, device=DEV)
    wide[:, :n] = t32(dy)
    dyv = wide[:, :n]
    assert dyv.stride(0) == n + pad
    xt, at, dt, bt = t32(x), t32(a), t32(d), t32(b)
    hc = F.new_h2cache(rows, n, DEV)
    F.acdc_forward(xt, at, dt, bt, h2cache=hc)
    g = [torch.zeros(n, device=DEV) for _ in range(3)]
    dx = F.acdc_backward(xt, dyv, at, dt, *g, accumulate=False, h2cache=hc)
    torch.cuda.synchronize()
    X, A, D, B, DY = (v.astype(np.float64) for v in (x, a, d, b, dy))
    _, h2 = O.acdc_forward(X, A, D, B)
    dxr, gar, gdr, gbr = O.acdc_backward(X, h2, DY, A, D)
    assert_close_rows(dx, dxr, n, "dx")
    for mine, ref, nm in zip(g, (gar, gdr, gbr), ("grad_a", "grad_d", "grad_bias")):
        assert_close_grad(mine, ref, n, rows, nm)
