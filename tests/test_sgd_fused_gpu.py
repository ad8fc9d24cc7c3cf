"""GPU tier: backward fused with the momentum-SGD step (acdc_bwd_sgd_f32;
reference AcdcLayer.backward + Sgd.step, layers.py:148-156, training.py:58-98).

Checked three ways: against the fp64 oracle (oracle.sgd_step on the oracle's
gradients), against the unfused path (backward "+=" then the _foreach Sgd.step)
on identical inputs, and end to end through train(fused_sgd=True)."""

import numpy as np
import pytest
import torch

from oracle import acdc_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda"


def f32(rng, *shape, mean=0.0, std=1.0):
    return (mean + std * rng.standard_normal(shape)).astype(np.float32)


def t(v):
    return torch.as_tensor(v, device=DEV)


@pytest.mark.parametrize("n,rows,cached", [(256, 64, False), (256, 64, True), (1024, 33, True), (16, 7, False),
                                           (4096, 40, True), (1, 5, False)])
def test_fused_step_matches_oracle(n, rows, cached):
    from paper_1511_05946_b200 import functional as F

    rng = np.random.default_rng(n + rows)
    x, dy = f32(rng, rows, n), f32(rng, rows, n)
    a, d, b = f32(rng, n, mean=1.0, std=0.3), f32(rng, n, mean=1.0, std=0.3), f32(rng, n, std=0.3)
    vel = [f32(rng, n, std=0.01) for _ in range(3)]
    old = [f32(rng, n, std=0.5) for _ in range(3)]  # gradients accumulated by an earlier backward
    lr, mu, wd = 0.05, 0.9, 1e-3
    lr3 = [lr * 1.0, lr * 0.5, lr * 2.0]
    wd3 = [wd, 0.0, wd]
    P = [t(v.copy()) for v in (a, d, b)]
    V = [t(v.copy()) for v in vel]
    G = [t(v.copy()) for v in old]
    hc = None
    if cached:
        hc = F.new_h2cache(rows, n, DEV)
        F.acdc_forward(t(x), P[0], P[1], P[2], h2cache=hc)
    dx = F.acdc_backward_sgd(t(x), t(dy), P, V, lr3, wd3, mu, grads=G, accumulate=True, h2cache=hc)
    torch.cuda.synchronize()
    # oracle: backward (+=) then the reference update
    X, DY = x.astype(np.float64), dy.astype(np.float64)
    A, D, B = (v.astype(np.float64) for v in (a, d, b))
    _, h2 = O.acdc_forward(X, A, D, B)
    grads = [v.astype(np.float64) for v in old]
    dxr, _, _, _ = O.acdc_backward(X, h2, DY, A, D, grads)
    vals, vels = [A.copy(), D.copy(), B.copy()], [v.astype(np.float64) for v in vel]
    full = [g.copy() for g in grads]
    for k in range(3):
        O.sgd_step(vals[k], grads[k], vels[k], lr, momentum=mu, weight_decay=wd, decay=wd3[k] != 0.0,
                   lr_mult=lr3[k] / lr)
    assert float(np.abs(dx.double().cpu().numpy() - dxr).max()) <= O.fp32_tolerance(n, dxr)
    for k in range(3):
        # the update inherits the gradient's error, scaled by lr
        gt = O.grad_tolerance(n, rows, full[k])
        tol_v = lr3[k] * gt + 4 * O.EPS32 * max(1.0, float(np.abs(vels[k]).max()))
        tol_p = tol_v + 4 * O.EPS32 * max(1.0, float(np.abs(vals[k]).max()))
        ev = float(np.abs(V[k].double().cpu().numpy() - vels[k]).max())
        ep = float(np.abs(P[k].double().cpu().numpy() - vals[k]).max())
        assert ev <= tol_v, (k, ev, tol_v)
        assert ep <= tol_p, (k, ep, tol_p)
        assert float(G[k].abs().max()) == 0.0  # zeroed like p.grad[...] = 0


def test_fused_step_equals_unfused_path():
    """Same dx bit for bit; parameters / velocities within fp32 rounding of
    backward(+=) followed by the _foreach Sgd.step."""
    from paper_1511_05946_b200 import AcdcLayer
    from paper_1511_05946_b200 import training as T

    n, rows = 512, 96
    rng = np.random.default_rng(5)
    x, dy = t(f32(rng, rows, n)), t(f32(rng, rows, n))
    layers = [AcdcLayer(n, device=DEV) for _ in range(2)]
    for L in layers:
        L.a.copy_(t(f32(rng, n, mean=1.0, std=0.2)))
        L.d.copy_(t(f32(rng, n, mean=1.0, std=0.2)))
        L.bias_d.copy_(t(f32(rng, n, std=0.2)))
    layers[1].a.copy_(layers[0].a)
    layers[1].d.copy_(layers[0].d)
    layers[1].bias_d.copy_(layers[0].bias_d)
    cfg = T.SgdConfig(learning_rate=0.02, momentum=0.9, weight_decay=1e-2)
    for L in layers:
        L.params()[2].decay = True  # exercise the decay flag and lr_mult
        L.params()[1].lr_mult = 0.5
    opts = [T.Sgd(L.params(), cfg) for L in layers]
    for step in range(3):
        y0, y1 = layers[0].forward(x), layers[1].forward(x)
        dx0 = layers[0].backward(dy)
        opts[0].step()
        dx1 = opts[1].backward_step(layers[1], dy)
        if step == 0:  # identical inputs: the same kernels give identical outputs
            assert torch.equal(y0, y1) and torch.equal(dx0, dx1)
        else:  # the parameters now differ by update rounding
            torch.testing.assert_close(dx1, dx0, rtol=1e-5, atol=1e-5)
        for p0, p1, v0, v1 in zip(layers[0].params(), layers[1].params(), opts[0].velocities, opts[1].velocities):
            torch.testing.assert_close(p1.value, p0.value, rtol=2e-6, atol=2e-7)
            torch.testing.assert_close(v1, v0, rtol=2e-6, atol=2e-7)
            assert float(p1.grad.abs().max()) == 0.0
    assert opts[1].step_count == 3


@pytest.mark.parametrize("fused_stack,n", [(True, 256), (False, 256), (True, 8192), (False, 16384)])
def test_cascade_backward_step(fused_stack, n):
    """n >= 8192: the fused stack's block backward reads the cascade's row-pair
    h2 layout, the per-layer path the half-length layer kernels."""
    from paper_1511_05946_b200 import AcdcLayer, Cascade, PermutationLayer, ReluLayer
    from paper_1511_05946_b200 import training as T

    rows, depth = 48, 3
    rng = np.random.default_rng(11)
    perms = [rng.permutation(n) for _ in range(depth)]
    init = [(f32(rng, n, mean=1.0, std=0.2), f32(rng, n, mean=1.0, std=0.2), f32(rng, n, std=0.1))
            for _ in range(depth)]

    def make():
        layers = []
        for i in range(depth):
            L = AcdcLayer(n, device=DEV)
            for dst, src in zip((L.a, L.d, L.bias_d), init[i]):
                dst.copy_(t(src))
            layers.append(L)
            if i < depth - 1:
                layers.append(ReluLayer(n, device=DEV))
                layers.append(PermutationLayer(n, perm=perms[i], device=DEV))
        c = Cascade(layers)
        if not fused_stack:
            c._fused = None  # force the per-layer path
        return c

    c0, c1 = make(), make()
    assert c0.fused == fused_stack
    cfg = T.SgdConfig(learning_rate=0.01, momentum=0.8)
    o0, o1 = T.Sgd(c0.params(), cfg), T.Sgd(c1.params(), cfg)
    x, dy = t(f32(rng, rows, n)), t(f32(rng, rows, n))
    for it in range(2):
        c0.forward(x)
        c1.forward(x)
        g0 = c0.backward(dy)
        o0.step()
        g1 = o1.backward_step(c1, dy)
        tol = 0 if it == 0 else 1e-5
        torch.testing.assert_close(g1, g0, rtol=tol, atol=tol)
        for p0, p1 in zip(c0.params(), c1.params()):
            torch.testing.assert_close(p1.value, p0.value, rtol=2e-6, atol=2e-7)


def test_train_fused_matches_reference(golden):
    """train(fused_sgd=True) reproduces the reference train() curve and final
    parameters (same golden vectors as tests/test_training.py)."""
    from paper_1511_05946_b200 import acdc_cascade
    from paper_1511_05946_b200 import training as T

    ds = T.make_regression(11, n_samples=256, n_in=64, n_out=64)
    casc = acdc_cascade(64, 2)
    cfg = T.SgdConfig(learning_rate=0.002, momentum=0.9, lr_decay_factor=0.5, lr_decay_every=12)
    curve = T.train(casc, ds, cfg, init_scheme=T.InitScheme(), epochs=4, batch_size=48, seed=1, fused_sgd=True)
    np.testing.assert_allclose(curve, golden["train_curve"], rtol=2e-4)
    got = np.stack([torch.cat([L.a, L.d, L.bias_d]).cpu().numpy() for L in casc.layers])
    np.testing.assert_allclose(got, golden["train_curve_params"], rtol=0, atol=2e-4)


def test_train_fused_matches_unfused():
    from paper_1511_05946_b200 import acdc_cascade
    from paper_1511_05946_b200 import training as T

    ds = T.make_regression(1, n_samples=256, n_in=256, n_out=256)
    cfg = T.SgdConfig(learning_rate=0.002, momentum=0.9)
    curves = []
    for fused in (False, True):
        c = acdc_cascade(256, 3, device=DEV)
        curves.append(T.train(c, ds, cfg, init_scheme=T.InitScheme(), epochs=3, batch_size=64, seed=2,
                              fused_sgd=fused))
    np.testing.assert_allclose(curves[1], curves[0], rtol=1e-5)
