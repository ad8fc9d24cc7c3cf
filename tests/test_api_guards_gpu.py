"""GPU tier: argument guards and edge cases on the public entry points.

* the fused cascade on an empty batch returns an empty (0, n) result like the
  reference (layers.py:336-344 iterate over zero rows), and its backward
  leaves the accumulated gradients unchanged;
* a backward whose grad_y has a different row count than the forward input
  raises ValueError (reference ``AcdcLayer.backward`` shapes, layers.py:148-156)
  instead of reading / writing out of bounds;
* caller-supplied ``out=`` / ``h2cache=`` tensors are validated;
* the SGD-fused reduction publishes the updated parameters before a
  programmatically-dependent backward of the same layer reads them;
* ``train`` accepts a bare layer, like the reference (training.py:210-249).
"""

import numpy as np
import pytest
import torch

from oracle import acdc_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _stack(n, depth, relu=True, perm=True, seed=0):
    from paper_1511_05946_b200 import AcdcLayer, Cascade, PermutationLayer, ReluLayer

    rng = np.random.default_rng(seed)
    layers = []
    for i in range(depth):
        L = AcdcLayer(n)
        L.a.copy_(torch.as_tensor(1 + 0.2 * rng.standard_normal(n), dtype=torch.float32))
        L.d.copy_(torch.as_tensor(1 + 0.2 * rng.standard_normal(n), dtype=torch.float32))
        layers.append(L)
        if i < depth - 1:
            if relu:
                layers.append(ReluLayer(n))
            if perm:
                layers.append(PermutationLayer(n, perm=rng.permutation(n)))
    return Cascade(layers)


def test_fused_cascade_empty_batch():
    casc = _stack(1024, 3)
    assert casc.fused
    y = casc.forward(torch.zeros(0, 1024, device=DEV))
    assert tuple(y.shape) == (0, 1024)
    before = [p.grad.clone() for p in casc.params()]
    dx = casc.backward(torch.zeros(0, 1024, device=DEV))
    assert tuple(dx.shape) == (0, 1024)
    for b, p in zip(before, casc.params()):
        assert torch.equal(b, p.grad)


def test_fused_cascade_grad_rows_mismatch():
    casc = _stack(512, 2)
    casc.forward(torch.randn(8, 512, device=DEV))
    with pytest.raises(ValueError, match="rows"):
        casc.backward(torch.randn(6, 512, device=DEV))
    casc.forward(torch.randn(8, 512, device=DEV))
    with pytest.raises(ValueError, match="rows"):
        casc.backward(torch.randn(10, 512, device=DEV))


def test_out_and_cache_validation():
    from paper_1511_05946_b200 import functional as F

    n = 1024
    x = torch.randn(6, n, device=DEV)
    v = torch.ones(n, device=DEV)
    g = [torch.zeros(n, device=DEV) for _ in range(3)]
    with pytest.raises(ValueError):
        F.acdc_forward(x, v, v, v, out=torch.empty(1, n, device=DEV))
    with pytest.raises(ValueError):
        F.acdc_forward(x, v, v, v, out=torch.empty(6, n, device=DEV, dtype=torch.float64))
    with pytest.raises(ValueError):
        F.acdc_forward(x, v, v, v, out=torch.empty(6, n))  # not on the device, not pinned
    small = F.new_h2cache(2, n, DEV)
    with pytest.raises(ValueError):
        F.acdc_forward(x, v, v, v, h2cache=small)
    with pytest.raises(ValueError):
        F.acdc_backward(x, x, v, v, *g, h2cache=small)
    with pytest.raises(ValueError):
        F.acdc_backward(x, x, v, v, *g, out=torch.empty(5, n, device=DEV))
    z = torch.randn(4, 256, dtype=torch.complex64, device=DEV)
    cv = torch.ones(256, dtype=torch.complex64, device=DEV)
    with pytest.raises(ValueError):
        F.afdf_forward(z, cv, cv, out=torch.empty(4, 256, device=DEV))
    # a correctly sized cache and out still work
    hc = F.new_h2cache(6, n, DEV)
    y = F.acdc_forward(x, v, v, torch.zeros(n, device=DEV), out=torch.empty(6, n, device=DEV), h2cache=hc)
    torch.cuda.synchronize()
    assert torch.allclose(y, x, atol=1e-4)  # identity layer


def test_sgd_fused_update_visible_to_next_backward():
    """A depth-1 fused cascade: backward(retain_cache, sgd) twice; the second
    backward must use the parameters the first one's SGD epilogue wrote."""
    from paper_1511_05946_b200 import functional as F

    n, rows = 1024, 64
    rng = np.random.default_rng(5)
    x = torch.as_tensor(rng.standard_normal((rows, n)), dtype=torch.float32, device=DEV)
    dy = torch.as_tensor(rng.standard_normal((rows, n)), dtype=torch.float32, device=DEV)
    a = torch.as_tensor(1 + 0.2 * rng.standard_normal(n), dtype=torch.float32, device=DEV)
    d = torch.as_tensor(1 + 0.2 * rng.standard_normal(n), dtype=torch.float32, device=DEV)
    b = torch.zeros(n, device=DEV)
    vel = [torch.zeros(n, device=DEV) for _ in range(3)]
    lr = (0.5, 0.5, 0.5)
    hc = F.new_h2cache(rows, n, DEV)
    F.acdc_forward(x, a, d, b, h2cache=hc)
    F.acdc_backward_sgd(x, dy, (a, d, b), vel, lr, (0.0, 0.0, 0.0), 0.0, h2cache=hc)
    dx2 = F.acdc_backward_sgd(x, dy, (a, d, b), vel, lr, (0.0, 0.0, 0.0), 0.0, h2cache=hc)
    torch.cuda.synchronize()
    # after two updates a, d hold the second step's values; dx2 was computed
    # with the values after the FIRST step, i.e. a - v2, d - v2 (p1 = p2 - v2)
    A = (a - vel[0]).double().cpu().numpy()
    D = (d - vel[1]).double().cpu().numpy()
    DY = dy.double().cpu().numpy()
    g3 = O.dct2_rows(DY)
    g1 = O.dct3_rows(g3 * D)
    ref = g1 * A
    err = float(np.abs(dx2.double().cpu().numpy() - ref).max())
    assert err <= O.fp32_tolerance(n, ref) * 4, err


def test_train_accepts_bare_layer():
    from paper_1511_05946_b200 import AcdcLayer
    from paper_1511_05946_b200.training import SgdConfig, make_regression, train

    ds = make_regression(0, n_samples=256, n_in=32, n_out=32)
    layer = AcdcLayer(32)
    losses = train(layer, ds, SgdConfig(learning_rate=0.01), epochs=2, batch_size=64)
    assert len(losses) == 2 and all(np.isfinite(losses))


@pytest.mark.parametrize("n", [100, 256])
def test_naive_mode_layer(n):
    """dct_mode="naive" (transforms.py:141, 152): any n, dense transforms;
    matches the fp64 oracle (and the fast layer where n is a power of two)."""
    from paper_1511_05946_b200 import AcdcLayer

    rng = np.random.default_rng(n)
    rows = 9
    L = AcdcLayer(n, dct_mode="naive")
    assert L.dct_plan.backend == "naive" and L.dct_plan.cos_matrix.shape == (n, n)
    a, d, b = 1 + 0.3 * rng.standard_normal(n), 1 + 0.3 * rng.standard_normal(n), 0.2 * rng.standard_normal(n)
    for t, v in ((L.a, a), (L.d, d), (L.bias_d, b)):
        t.copy_(torch.as_tensor(v, dtype=torch.float32))
    x, dy = rng.standard_normal((rows, n)).astype(np.float32), rng.standard_normal((rows, n)).astype(np.float32)
    y = L.forward(x)  # host in -> fp64 numpy out
    dx = L.backward(dy)
    A, D, B = (t.double().cpu().numpy() for t in (L.a, L.d, L.bias_d))
    C = O.dct_matrix(n)
    h2 = (x * A) @ C
    yr = (h2 * D + B) @ C.T
    g3 = dy.astype(np.float64) @ C
    g1 = (g3 * D) @ C.T
    assert np.abs(y - yr).max() <= 4 * O.fp32_tolerance(n, yr)
    assert np.abs(dx - g1 * A).max() <= 4 * O.fp32_tolerance(n, g1 * A)
    for mine, ref in ((L.grad_bias_d, g3.sum(0)), (L.grad_d, (h2 * g3).sum(0)), (L.grad_a, (x * g1).sum(0))):
        assert np.abs(mine.double().cpu().numpy() - ref).max() <= 4 * O.grad_tolerance(n, rows, ref)
    if n == 256:
        F_ = AcdcLayer(n)
        for t, v in ((F_.a, a), (F_.d, d), (F_.bias_d, b)):
            t.copy_(torch.as_tensor(v, dtype=torch.float32))
        assert np.abs(F_.forward(x) - y).max() <= 4 * O.fp32_tolerance(n, yr)
    from paper_1511_05946_b200 import AfdfLayer

    assert AfdfLayer(64).fft_plan.twiddle.shape == (32,)


@pytest.mark.parametrize("n,rows,cplx", [(7, 5, False), (1000, 33, True), (32768, 3, True), (16384, 4, False)])
def test_relu_perm_native_layers(n, rows, cplx):
    """ReluLayer / PermutationLayer outside the fused cascade run the native
    kernels (layers.py:218-265): strict mask, gather by perm, scatter by
    argsort(perm); complex rows permute as 8-byte elements."""
    from paper_1511_05946_b200 import PermutationLayer, ReluLayer

    rng = np.random.default_rng(n)
    p = rng.permutation(n)
    x = rng.standard_normal((rows, n)).astype(np.float32)
    x[0, : min(n, 3)] = 0.0  # exact zeros: masked (strict x > 0)
    if cplx:
        xc = (x + 1j * rng.standard_normal((rows, n))).astype(np.complex64)
        P = PermutationLayer(n, perm=p)
        y = P.forward(torch.as_tensor(xc, device=DEV))
        assert torch.equal(y.cpu(), torch.as_tensor(xc)[:, p])
        g = P.backward(y)
        assert torch.equal(g.cpu(), torch.as_tensor(xc))
        return
    R = ReluLayer(n)
    y = R.forward(torch.as_tensor(x, device=DEV))
    assert torch.equal(y.cpu(), torch.as_tensor(np.where(x > 0, x, 0.0).astype(np.float32)))
    dy = rng.standard_normal((rows, n)).astype(np.float32)
    dx = R.backward(torch.as_tensor(dy, device=DEV))
    assert torch.equal(dx.cpu(), torch.as_tensor(np.where(x > 0, dy, 0.0).astype(np.float32)))
    P = PermutationLayer(n, perm=p)
    yp = P.forward(torch.as_tensor(x, device=DEV))
    assert torch.equal(yp.cpu(), torch.as_tensor(x[:, p]))
    assert torch.equal(P.backward(yp).cpu(), torch.as_tensor(x))
