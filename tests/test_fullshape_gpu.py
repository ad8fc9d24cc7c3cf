"""GPU tier: parity at the exact BASELINE.json shapes, through the same layer
API the bench times, against the reference's OWN compiled CPU kernels
(``oracle/_ref``: ``_kernels.pyx`` built from /root/reference, fp64, driven
with the reference layer call sequence by ``oracle/ref_kernels.py``).

* M   single ACDC layer N=4096, B=16384 — h2-cache (TMEM backward) and
      recompute modes (layers.py:141-156)
* S   the size sweep N=128..32768 at B=16384 (configs[1])
* C3  12 blocks ACDC+ReLU+Perm, N=1024, B=8192, fused cascade (layers.py:309-357)
* C4  32 ACDC layers, N=4096, B=4096 per GPU, one training step with the
      momentum-SGD update fused into each block's gradient reduction
      (training.py:58-98)
* C5  AFDF N=8192 complex64, 8192 rows (one GPU's shard of 65536 over 8)

Tolerances (oracle/acdc_oracle.py): rows max-abs <=
4 log2N eps32 max(rms, 1); parameter grads <= 4 (log2N + log2B) eps32
max(|ref|, 1).  Stacks multiply the per-block bound by ``chain_factor`` of
the blocks' rms gains (each block adds its own rounding and passes the
incoming error on through rms(a) rms(d); ReLU / Perm add no gain); a
layer's gradient reduction reads x_l and dy_l, which carry the rounding of
every other block, so its bound is scaled by the chain over all blocks.

Large arrays are checked in row chunks (the reference runs on all host
threads) so host memory stays bounded at N=32768.
"""

import numpy as np
import pytest
import torch

from oracle import acdc_oracle as O
from oracle import ref_kernels as R

pytestmark = pytest.mark.gpu
DEV = "cuda"
CHUNK = 2048


@pytest.fixture(scope="module", autouse=True)
def _need_ref():
    if R.load() is None:
        pytest.skip("oracle/_ref (the reference's compiled kernels) is not built")


def _gauss(gen, *shape, mean=0.0, std=1.0):
    return mean + std * torch.randn(*shape, device=DEV, generator=gen)


def _err(mine, ref):
    return float(np.abs(np.asarray(mine, dtype=np.float64) - ref).max()) if ref.size else 0.0


def _layer_vs_ref(n, rows, cache_h2, seed):
    """AcdcLayer forward+backward on the GPU vs the reference kernels, chunked."""
    from paper_1511_05946_b200 import AcdcLayer

    g = torch.Generator(device=DEV)
    g.manual_seed(seed)
    layer = AcdcLayer(n, device=DEV, cache_h2=cache_h2)
    layer.a.copy_(_gauss(g, n, mean=1.0, std=0.4))
    layer.d.copy_(_gauss(g, n, mean=1.0, std=0.4))
    layer.bias_d.copy_(_gauss(g, n, std=0.3))
    x = _gauss(g, rows, n)
    dy = _gauss(g, rows, n)
    y = layer.forward(x)
    dx = layer.backward(dy)
    torch.cuda.synchronize()
    a, d, b = (t.double().cpu().numpy() for t in (layer.a, layer.d, layer.bias_d))
    ref = R.RefAcdc(a, d, b)
    thr = R.threads_available()
    gsum = [np.zeros(n) for _ in range(3)]
    worst = {"y": 0.0, "dx": 0.0}
    for lo in range(0, rows, CHUNK):
        hi = min(rows, lo + CHUNK)
        xc = x[lo:hi].double().cpu().numpy()
        dyc = dy[lo:hi].double().cpu().numpy()
        yr, dxr, ga, gd, gb = R.fwd_bwd_threaded(ref, xc, dyc, thr)
        for k, v in enumerate((ga, gd, gb)):
            gsum[k] += v
        for name, mine, r in (("y", y[lo:hi], yr), ("dx", dx[lo:hi], dxr)):
            e = _err(mine.double().cpu().numpy(), r)
            tol = O.fp32_tolerance(n, r)
            assert e <= tol, f"{name} rows [{lo},{hi}): {e:.3e} > {tol:.3e} (N={n}, B={rows})"
            worst[name] = max(worst[name], e / tol)
    for name, mine, r in (("grad_a", layer.grad_a, gsum[0]), ("grad_d", layer.grad_d, gsum[1]),
                          ("grad_bias", layer.grad_bias_d, gsum[2])):
        e = _err(mine.double().cpu().numpy(), r)
        tol = O.grad_tolerance(n, rows, r)
        assert e <= tol, f"{name}: {e:.3e} > {tol:.3e} (N={n}, B={rows})"
        worst[name] = e / tol
    return worst


@pytest.mark.parametrize("cache_h2", [True, False], ids=["h2cache", "recompute"])
def test_metric_shape(cache_h2):
    """BASELINE metric: N=4096, B=16384 — the exact kernels bench.py times."""
    w = _layer_vs_ref(4096, 16384, cache_h2, seed=11)
    print("err/tol", w)


@pytest.mark.parametrize("n", [1 << k for k in range(7, 16)])
def test_sweep_full_batch(n):
    """configs[1]: every sweep size at B=16384 (default mode: h2 cache where supported)."""
    w = _layer_vs_ref(n, 16384, True, seed=n)
    print("err/tol", n, w)


def _ckpt_masks(casc, rows, n, depth, perms, relu_after):
    from paper_1511_05946_b200 import functional as F

    xs, _ = F._ckpt_views(casc._cache[1], rows, n, depth)
    masks = []
    for l in range(depth - 1):
        if not relu_after[l]:
            masks.append(None)
            continue
        xn = xs[l].cpu().numpy()  # x_{l+1} = perm(relu(u_l))
        masks.append((xn[:, np.argsort(perms[l])] if perms[l] is not None else xn) > 0)
    return masks


def test_c3_cascade_full_batch():
    """C3: 12 blocks ACDC+ReLU+Perm, N=1024, B=8192, fused on-chip cascade."""
    from paper_1511_05946_b200 import AcdcLayer, Cascade, PermutationLayer, ReluLayer

    n, depth, rows = 1024, 12, 8192
    rng = np.random.default_rng(3)
    g = torch.Generator(device=DEV)
    g.manual_seed(3)
    layers, acdc, perms = [], [], []
    for i in range(depth):
        L = AcdcLayer(n, device=DEV)
        L.a.copy_(_gauss(g, n, mean=1.0, std=0.2))
        L.d.copy_(_gauss(g, n, mean=1.0, std=0.2))
        L.bias_d.copy_(_gauss(g, n, std=0.1))
        layers.append(L)
        acdc.append(L)
        if i < depth - 1:
            p = rng.permutation(n)
            perms.append(p)
            layers += [ReluLayer(n, device=DEV), PermutationLayer(n, perm=p, device=DEV)]
    casc = Cascade(layers)
    assert casc.fused
    x = _gauss(g, rows, n)
    dy = _gauss(g, rows, n)
    y = casc.forward(x)
    dx = casc.backward(dy, retain_cache=True)
    torch.cuda.synchronize()
    masks = _ckpt_masks(casc, rows, n, depth, perms, [True] * (depth - 1))
    thr = R.threads_available()
    refs = [R.RefAcdc(*(t.double().cpu().numpy() for t in (L.a, L.d, L.bias_d))) for L in acdc]
    gains = [O.block_gain(r.a, r.d) for r in refs]
    # forward (reference kernels per block; ReLU with the GPU's masks; Perm gather)
    h = x.double().cpu().numpy()
    xs, h2s = [], []
    for l, r in enumerate(refs):
        xs.append(h)
        u, h2 = r.forward(h) if thr == 1 else _threaded(r.forward, h, thr)
        h2s.append(h2)
        if l < depth - 1:
            u = np.where(masks[l], u, 0.0)
            u = u[:, perms[l]]
        h = u
    yr = h
    tol_y = O.chain_factor(gains) * O.fp32_tolerance(n, yr)
    e = _err(y.double().cpu().numpy(), yr)
    assert e <= tol_y, f"C3 y: {e:.3e} > {tol_y:.3e}"
    # backward, last block first
    gcur = dy.double().cpu().numpy()
    grads = [None] * depth
    for l in range(depth - 1, -1, -1):
        r = refs[l]
        dxl, ga, gd, gb = _threaded_bwd(r, xs[l], h2s[l], gcur, thr)
        grads[l] = (ga, gd, gb)
        if l > 0:
            dxl = dxl[:, np.argsort(perms[l - 1])]
            dxl = np.where(masks[l - 1], dxl, 0.0)
        gcur = dxl
    tol_dx = O.chain_factor(gains[::-1]) * O.fp32_tolerance(n, gcur)
    e = _err(dx.double().cpu().numpy(), gcur)
    assert e <= tol_dx, f"C3 dx: {e:.3e} > {tol_dx:.3e}"
    chain_all = O.chain_factor(gains)
    for l, (L, (ga, gd, gb)) in enumerate(zip(acdc, grads)):
        for name, mine, r in (("grad_a", L.grad_a, ga), ("grad_d", L.grad_d, gd), ("grad_bias", L.grad_bias_d, gb)):
            tol = chain_all * O.grad_tolerance(n, rows, r)
            e = _err(mine.double().cpu().numpy(), r)
            assert e <= tol, f"C3 block {l} {name}: {e:.3e} > {tol:.3e}"


def _threaded(fn, h, thr):
    from concurrent.futures import ThreadPoolExecutor

    b = np.linspace(0, h.shape[0], thr + 1).astype(int)
    with ThreadPoolExecutor(thr) as ex:
        parts = list(ex.map(lambda i: fn(h[b[i]:b[i + 1]]), range(thr)))
    return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])


def _threaded_bwd(r, x, h2, dy, thr):
    from concurrent.futures import ThreadPoolExecutor

    b = np.linspace(0, x.shape[0], thr + 1).astype(int)
    with ThreadPoolExecutor(thr) as ex:
        parts = list(ex.map(lambda i: r.backward(x[b[i]:b[i + 1]], h2[b[i]:b[i + 1]], dy[b[i]:b[i + 1]]),
                            range(thr)))
    return (np.concatenate([p[0] for p in parts]), sum(p[1] for p in parts), sum(p[2] for p in parts),
            sum(p[3] for p in parts))


def test_c4_deep_sell_fused_sgd_step():
    """C4: 32 ACDC layers N=4096, B=4096 rows (one GPU's batch), one training
    step with the SGD update fused into each block's reduction: dx, and the
    velocity v = -lr * grad each layer's update applied (training.py:72-84)."""
    from paper_1511_05946_b200 import acdc_cascade
    from paper_1511_05946_b200.training import Sgd, SgdConfig

    n, depth, rows, lr = 4096, 32, 4096, 1e-3
    g = torch.Generator(device=DEV)
    g.manual_seed(4)
    casc = acdc_cascade(n, depth, device=DEV)
    assert casc.fused
    for L in casc.layers:
        L.a.copy_(_gauss(g, n, mean=1.0, std=0.061))
        L.d.copy_(_gauss(g, n, mean=1.0, std=0.061))
        L.bias_d.copy_(_gauss(g, n, std=0.01))
    refs = [R.RefAcdc(*(t.double().cpu().numpy() for t in (L.a, L.d, L.bias_d))) for L in casc.layers]
    x = _gauss(g, rows, n)
    dy = _gauss(g, rows, n)
    opt = Sgd(casc.params(), SgdConfig(learning_rate=lr, momentum=0.9))
    y = casc.forward(x)
    dx = opt.backward_step(casc, dy)
    torch.cuda.synchronize()
    thr = R.threads_available()
    gains = [O.block_gain(r.a, r.d) for r in refs]
    h = x.double().cpu().numpy()
    xs, h2s = [], []
    for r in refs:
        xs.append(h)
        h, h2 = _threaded(r.forward, h, thr)
        h2s.append(h2)
    e = _err(y.double().cpu().numpy(), h)
    tol = O.chain_factor(gains) * O.fp32_tolerance(n, h)
    assert e <= tol, f"C4 y: {e:.3e} > {tol:.3e}"
    gcur = dy.double().cpu().numpy()
    grads = [None] * depth
    for l in range(depth - 1, -1, -1):
        gcur, ga, gd, gb = _threaded_bwd(refs[l], xs[l], h2s[l], gcur, thr)
        grads[l] = (ga, gd, gb)
    e = _err(dx.double().cpu().numpy(), gcur)
    tol = O.chain_factor(gains[::-1]) * O.fp32_tolerance(n, gcur)
    assert e <= tol, f"C4 dx: {e:.3e} > {tol:.3e}"
    chain_all = O.chain_factor(gains)
    vel = opt.velocities
    for l in range(depth):
        for k, name in enumerate(("a", "d", "bias_d")):
            ref_v = -lr * grads[l][k]
            mine = vel[3 * l + k].double().cpu().numpy()
            tol = lr * chain_all * O.grad_tolerance(n, rows, grads[l][k])
            e = _err(mine, ref_v)
            assert e <= tol, f"C4 layer {l} velocity {name}: {e:.3e} > {tol:.3e}"
        for p in casc.layers[l].params():  # the fused step zeroes the accumulated grads
            assert float(p.grad.abs().max()) == 0.0


def test_c5_afdf_shard():
    """C5: AFDF N=8192 complex64, 8192 rows (65536 over 8 GPUs, one shard)."""
    from paper_1511_05946_b200 import AfdfLayer

    n, rows = 8192, 8192
    g = torch.Generator(device=DEV)
    g.manual_seed(5)
    cg = lambda *s, m=0.0, sd=1.0: torch.complex(_gauss(g, *s, mean=m, std=sd), _gauss(g, *s, std=sd))
    layer = AfdfLayer(n, device=DEV)
    layer.a.copy_(cg(n, m=1.0, sd=0.1))
    layer.d.copy_(cg(n, m=1.0, sd=0.1))
    x, dy = cg(rows, n), cg(rows, n)
    y = layer.forward(x)
    dx = layer.backward(dy)
    torch.cuda.synchronize()
    a, d = layer.a.cpu().numpy().astype(np.complex128), layer.d.cpu().numpy().astype(np.complex128)
    thr = R.threads_available()
    X, DY = x.cpu().numpy().astype(np.complex128), dy.cpu().numpy().astype(np.complex128)
    yr, dxr, gar, gdr = R.afdf_fwd_bwd_threaded(X, DY, a, d, thr)
    for name, mine, r in (("y", y, yr), ("dx", dx, dxr)):
        e = _err_c(mine, r)
        tol = O.fp32_tolerance(n, r)
        assert e <= tol, f"C5 {name}: {e:.3e} > {tol:.3e}"
    for name, mine, r in (("grad_a", layer.grad_a, gar), ("grad_d", layer.grad_d, gdr)):
        e = _err_c(mine, r)
        tol = O.grad_tolerance(n, rows, r)
        assert e <= tol, f"C5 {name}: {e:.3e} > {tol:.3e}"


def _err_c(mine, ref):
    return float(np.abs(mine.cpu().numpy().astype(np.complex128) - ref).max())
