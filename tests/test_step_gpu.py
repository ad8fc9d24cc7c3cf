"""GPU tier: the fused small-batch step (acdc_step_f32: forward + backward +
gradient reduction in one launch) vs the fp64 oracle and vs the separate
forward / backward kernels (layers.py:141-156).

Tolerances as tests/test_parity_gpu.py.  The step runs one
cluster of up to 8 CTAs (gradients summed over distributed shared memory), so
the cases cover one CTA, several CTAs, a full cluster and several row pairs
per group."""

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
    mine = mine.detach().cpu().double().numpy()
    tol = O.fp32_tolerance(n, ref)
    err = float(np.abs(mine - ref).max()) if ref.size else 0.0
    assert err <= tol, f"{what}: max err {err:.3e} > tol {tol:.3e} (N={n})"


def assert_close_grad(mine, ref, n, rows, what):
    mine = mine.detach().cpu().double().numpy()
    tol = O.grad_tolerance(n, rows, ref)
    err = float(np.abs(mine - ref).max())
    assert err <= tol, f"{what}: max err {err:.3e} > tol {tol:.3e} (N={n}, B={rows})"


def _inputs(n, rows, seed):
    rng = np.random.default_rng(seed)
    a, d = f32(rng, n, mean=1.0, std=0.4), f32(rng, n, mean=1.0, std=0.4)
    b = f32(rng, n, std=0.3)
    x, dy = f32(rng, rows, n), f32(rng, rows, n)
    return x, dy, a, d, b


def _rows_case(n, k):
    """Row counts relative to the fused limit: one pair, ragged, one CTA, several CTAs, the full cluster."""
    from paper_1511_05946_b200 import functional as F

    m = F.step_max_rows(n)
    return [1, 2, 3, 33 if m > 33 else m - 1, m // 2 + 1, m - 1, m][k]


@pytest.mark.parametrize("n", [256, 512, 1024, 2048])
@pytest.mark.parametrize("k", range(7))
def test_step_vs_oracle(n, k):
    from paper_1511_05946_b200 import functional as F

    rows = _rows_case(n, k)
    assert 0 < rows <= F.step_max_rows(n), "the case must run the fused kernel"
    x, dy, a, d, b = _inputs(n, rows, 7000 + n + rows)
    grads = [torch.zeros(n, device=DEV) for _ in range(3)]
    y, dx = F.acdc_step(t32(x), t32(dy), t32(a), t32(d), t32(b), *grads, accumulate=True)
    torch.cuda.synchronize()
    X, A, D, Bb, DY = (v.astype(np.float64) for v in (x, a, d, b, dy))
    yr, h2 = O.acdc_forward(X, A, D, Bb)
    dxr, gar, gdr, gbr = O.acdc_backward(X, h2, DY, A, D)
    assert_close_rows(y, yr, n, "y")
    assert_close_rows(dx, dxr, n, "dx")
    assert_close_grad(grads[0], gar, n, rows, "grad_a")
    assert_close_grad(grads[1], gdr, n, rows, "grad_d")
    assert_close_grad(grads[2], gbr, n, rows, "grad_bias")


@pytest.mark.parametrize("n,rows", [(256, 64), (256, 33), (512, 32), (1024, 16), (2048, 8)])
def test_step_vs_separate(n, rows):
    """The same formulas as the separate kernels; the grouping of the gradient
    partial sums differs (CTA sizes)."""
    from paper_1511_05946_b200 import functional as F

    x, dy, a, d, b = map(t32, _inputs(n, rows, 9100 + n))
    g1 = [torch.full((n,), 0.25, device=DEV) for _ in range(3)]
    g2 = [g.clone() for g in g1]
    y1, dx1 = F.acdc_step(x, dy, a, d, b, *g1, accumulate=True)
    y2 = F.acdc_forward(x, a, d, b)
    dx2 = F.acdc_backward(x, dy, a, d, *g2, accumulate=True)
    torch.cuda.synchronize()
    # same per-element formulas; the compiler's fma contraction may differ between kernels, and from
    # n = 1024 the separate path runs the half-length plan
    assert float((dx1 - dx2).abs().max()) <= O.fp32_tolerance(n, dx2.double().cpu().numpy())
    for u, v in zip(g1, g2):
        gt = O.grad_tolerance(n, rows, v.double().cpu().numpy())
        assert float((u - v).abs().max()) <= gt
    tol = O.fp32_tolerance(n, y2.double().cpu().numpy())
    assert float((y1 - y2).abs().max()) <= tol  # (the forward kernel's exchange layout may differ)


def test_step_accumulate_and_overwrite():
    from paper_1511_05946_b200 import functional as F

    n, rows = 256, 128
    x, dy, a, d, b = map(t32, _inputs(n, rows, 42))
    g = [torch.zeros(n, device=DEV) for _ in range(3)]
    F.acdc_step(x, dy, a, d, b, *g, accumulate=False)
    once = [v.clone() for v in g]
    F.acdc_step(x, dy, a, d, b, *g, accumulate=True)  # layers.py:152-155 "+="
    for u, v in zip(g, once):
        assert torch.allclose(u, 2 * v, rtol=1e-6, atol=1e-6)
    F.acdc_step(x, dy, a, d, b, *g, accumulate=False)
    for u, v in zip(g, once):
        assert torch.equal(u, v)  # deterministic


def test_step_empty_and_fallback():
    from paper_1511_05946_b200 import functional as F

    n = 256
    _, _, a, d, b = map(t32, _inputs(n, 1, 3))
    g = [torch.ones(n, device=DEV) for _ in range(3)]
    y, dx = F.acdc_step(torch.zeros(0, n, device=DEV), torch.zeros(0, n, device=DEV), a, d, b, *g, accumulate=True)
    torch.cuda.synchronize()
    assert y.shape == (0, n) and dx.shape == (0, n)
    assert all(torch.equal(v, torch.ones(n, device=DEV)) for v in g)
    F.acdc_step(torch.zeros(0, n, device=DEV), torch.zeros(0, n, device=DEV), a, d, b, *g, accumulate=False)
    torch.cuda.synchronize()
    assert all(float(v.abs().max()) == 0.0 for v in g)
    # above the fused limit: the separate kernels, same results as the oracle
    rows = F.step_max_rows(n) + 5
    x, dy, a2, d2, b2 = _inputs(n, rows, 5)
    gg = [torch.zeros(n, device=DEV) for _ in range(3)]
    y, dx = F.acdc_step(t32(x), t32(dy), t32(a2), t32(d2), t32(b2), *gg)
    X, A, D, Bb, DY = (v.astype(np.float64) for v in (x, a2, d2, b2, dy))
    yr, h2 = O.acdc_forward(X, A, D, Bb)
    dxr, gar, _, _ = O.acdc_backward(X, h2, DY, A, D)
    assert_close_rows(y, yr, n, "y")
    assert_close_rows(dx, dxr, n, "dx")
    assert_close_grad(gg[0], gar, n, rows, "grad_a")


def test_step_one_launch():
    """The fused step is one kernel: a CUDA graph of it holds one kernel node."""
    from paper_1511_05946_b200 import functional as F

    n, rows = 256, 128
    x, dy, a, d, b = map(t32, _inputs(n, rows, 11))
    g = [torch.zeros(n, device=DEV) for _ in range(3)]
    y, dx = torch.empty_like(x), torch.empty_like(x)
    F.prepare(n, x.device)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        F.acdc_step(x, dy, a, d, b, *g, accumulate=False, out_y=y, out_dx=dx)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        F.acdc_step(x, dy, a, d, b, *g, accumulate=False, out_y=y, out_dx=dx)
    ref = y.clone()
    y.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
