"""GPU tier: fused ACDC cascade (ACDC [+ReLU] [+Perm] blocks; layers.py:309-357)
vs the fp64 oracle and the reference golden cascades.

A ReLU whose fp64 pre-activation is within fp32 rounding of 0 may legitimately
take the other side on the GPU; the oracle backward therefore reuses the GPU's
masks (read from the fused forward's checkpoints), so the comparison checks the
arithmetic, not that sign coin-flip."""

import numpy as np
import pytest
import torch

from oracle import acdc_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda"


def f32(rng, *shape, mean=0.0, std=1.0):
    return (mean + std * rng.standard_normal(shape)).astype(np.float32)


def close(mine, ref, tol, what):
    mine = mine.detach().cpu().double().numpy() if isinstance(mine, torch.Tensor) else mine
    err = float(np.abs(mine - ref).max())
    assert err <= tol, f"{what}: {err:.3e} > {tol:.3e}"


def build(n, depth, rng, relu=True, perm=True, std=0.2):
    from paper_1511_05946_b200 import AcdcLayer, Cascade, PermutationLayer, ReluLayer

    layers, specs = [], []
    for i in range(depth):
        L = AcdcLayer(n)
        a, d, b = f32(rng, n, mean=1.0, std=std), f32(rng, n, mean=1.0, std=std), f32(rng, n, std=0.1)
        L.a.copy_(torch.as_tensor(a))
        L.d.copy_(torch.as_tensor(d))
        L.bias_d.copy_(torch.as_tensor(b))
        layers.append(L)
        specs.append({"kind": "acdc", "a": a.astype(np.float64), "d": d.astype(np.float64), "bias": b.astype(np.float64)})
        if i < depth - 1:
            if relu:
                layers.append(ReluLayer(n))
                specs.append({"kind": "relu"})
            if perm:
                pl = PermutationLayer(n, perm=rng.permutation(n))
                layers.append(pl)
                specs.append({"kind": "perm", "perm": pl.perm})
    return Cascade(layers), layers, specs


def oracle_with_masks(x, dy, specs, casc, rows):
    """fp64 forward; backward with the ReLU masks the GPU used."""
    from paper_1511_05946_b200 import functional as F

    y, caches = O.cascade_forward(x, specs)
    ckpt = casc._cache[1]
    n = x.shape[1]
    depth = sum(1 for s in specs if s["kind"] == "acdc")
    xs, _ = F._ckpt_views(ckpt, rows, n, depth)
    blk = -1
    for i, s in enumerate(specs):
        if s["kind"] == "acdc":
            blk += 1
        elif s["kind"] == "relu":
            xn = xs[blk].double().cpu().numpy()  # x_{blk+1} = perm(relu(u)) or relu(u)
            nxt = specs[i + 1] if i + 1 < len(specs) else None
            if nxt is not None and nxt["kind"] == "perm":
                caches[i] = xn[:, np.argsort(nxt["perm"])] > 0
            else:
                caches[i] = xn > 0
    dx, grads = O.cascade_backward(dy, specs, caches)
    return y, dx, [g for g in grads if g is not None]


@pytest.mark.parametrize("n,depth,rows,relu,perm", [(256, 3, 5, True, True), (1024, 12, 64, True, True),
                                                    (1024, 4, 33, False, True), (4096, 3, 16, True, False),
                                                    (512, 1, 7, False, False), (8192, 2, 5, True, True),
                                                    (16384, 2, 3, True, False)])
def test_fused_cascade_vs_oracle(n, depth, rows, relu, perm):
    rng = np.random.default_rng(n * 7 + depth)
    casc, layers, specs = build(n, depth, rng, relu, perm)
    assert casc.fused
    x, dy = f32(rng, rows, n), f32(rng, rows, n)
    y = casc.forward(torch.as_tensor(x, device=DEV))
    dx = casc.backward(torch.as_tensor(dy, device=DEV), retain_cache=True)
    torch.cuda.synchronize()
    yr, dxr, grads = oracle_with_masks(x.astype(np.float64), dy.astype(np.float64), specs, casc, rows)
    tol_rows = 4 * depth * O.fp32_tolerance(n, yr)
    close(y, yr, tol_rows, "y")
    close(dx, dxr, 4 * depth * O.fp32_tolerance(n, dxr), "dx")
    acdc = [l for l in layers if hasattr(l, "grad_bias_d")]
    for i, (L, (ga, gd, gb)) in enumerate(zip(acdc, grads)):
        close(L.grad_a, ga, depth * O.grad_tolerance(n, rows, ga), f"L{i} grad_a")
        close(L.grad_d, gd, depth * O.grad_tolerance(n, rows, gd), f"L{i} grad_d")
        close(L.grad_bias_d, gb, depth * O.grad_tolerance(n, rows, gb), f"L{i} grad_bias")


def test_fused_cascade_golden(golden):
    p = "casc_N256_K3_B2_"
    from paper_1511_05946_b200 import AcdcLayer, Cascade, PermutationLayer, ReluLayer

    layers = []
    for i in range(3):
        L = AcdcLayer(256)
        for nm in ("a", "d", "bias_d"):
            getattr(L, nm).copy_(torch.as_tensor(golden[p + f"L{i}_{nm}"], dtype=torch.float32))
        layers.append(L)
        if i < 2:
            layers += [ReluLayer(256), PermutationLayer(256, perm=golden[p + f"P{i}_perm"])]
    casc = Cascade(layers)
    assert casc.fused
    y = casc.forward(golden[p + "x"])  # host in -> host out, like the reference
    close(y, golden[p + "y"], 12 * O.fp32_tolerance(256, golden[p + "y"]), "golden y")
    dx = casc.backward(golden[p + "dy"])
    close(dx, golden[p + "dx"], 12 * O.fp32_tolerance(256, golden[p + "dx"]), "golden dx")
    for i, L in enumerate([l for l in layers if hasattr(l, "grad_bias_d")]):
        ref = golden[p + f"L{i}_grad_a"]
        close(L.grad_a, ref, 3 * O.grad_tolerance(256, 2, ref), f"golden L{i} grad_a")
    with pytest.raises(RuntimeError):
        casc.backward(golden[p + "dy"])


def test_fused_matches_unfused():
    """Fused kernels vs the per-layer path on the same fp32 parameters."""
    from paper_1511_05946_b200 import Cascade

    rng = np.random.default_rng(5)
    casc, layers, _ = build(1024, 5, rng)
    x = torch.as_tensor(f32(rng, 40, 1024), device=DEV)
    dy = torch.as_tensor(f32(rng, 40, 1024), device=DEV)
    y1 = casc.forward(x)
    dx1 = casc.backward(dy)
    g1 = [l.grad_a.clone() for l in layers if hasattr(l, "grad_bias_d")]
    for l in layers:
        l.zero_grads()
    unf = Cascade(layers)
    unf._fused = None  # force the per-layer path
    y2 = unf.forward(x)
    dx2 = unf.backward(dy)
    g2 = [l.grad_a.clone() for l in layers if hasattr(l, "grad_bias_d")]
    torch.testing.assert_close(y1, y2, rtol=1e-5, atol=1e-5)
    torch.testing.assert_close(dx1, dx2, rtol=1e-4, atol=1e-4)
    for u, v in zip(g1, g2):
        torch.testing.assert_close(u, v, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("n,depth,rows,relu,perm", [(256, 3, 9, True, True), (1024, 12, 130, True, True),
                                                    (2048, 4, 64, False, True), (4096, 3, 40, True, False)])
def test_deferred_reduction_matches_per_block(n, depth, rows, relu, perm):
    """The deferred form (block partials, one multi-block reduction at the end)
    is bit-identical to one reduction per block (forced by a per-layer hook),
    with accumulation into existing gradients, for the scatter (n=256) and the
    gather (512 <= n <= 8192) epilogues."""
    from paper_1511_05946_b200 import _lib

    rng = np.random.default_rng(7)
    casc, layers, _ = build(n, depth, rng, relu=relu, perm=perm)
    assert casc._fused is not None
    assert _lib.load().cascade_defer_ws_bytes(rows, n) > 0
    x = torch.as_tensor(f32(rng, rows, n), device=DEV)
    dy = torch.as_tensor(f32(rng, rows, n), device=DEV)
    acdc = [L for L in layers if hasattr(L, "grad_a")]
    res = []
    for hook in (None, lambda layer: None):
        for L in acdc:  # accumulate onto a nonzero starting gradient
            for g in (L.grad_a, L.grad_d, L.grad_bias_d):
                g.fill_(0.25)
        casc.forward(x)
        dx = casc.backward(dy, on_layer=hook)
        torch.cuda.synchronize()
        res.append([dx.clone()] + [g.clone() for L in acdc for g in (L.grad_a, L.grad_d, L.grad_bias_d)])
    for a_, b_ in zip(*res):
        assert torch.equal(a_, b_)


def test_deferred_reduction_abi_errors():
    from paper_1511_05946_b200 import _lib

    lib = _lib.load()
    assert lib.cascade_defer_ws_bytes(64, 128) == 0  # below the fused cascade's sizes
    assert lib.cascade_defer_ws_bytes(0, 1024) == 0
    assert lib.cascade_grad_reduce_f32(None, 0, 0, 0, 1024, None, 0, None) == 0  # nothing to reduce
    assert lib.cascade_grad_reduce_f32(None, 1 << 20, 2, 64, 1000, None, 0, None) != 0  # not a power of two


@pytest.mark.parametrize("n,depth,rows,relu,perm", [(512, 2, 6, True, True), (1024, 12, 130, True, True),
                                                    (1024, 4, 1, True, True), (512, 3, 2, True, True),
                                                    (1024, 5, 33, True, True), (2048, 3, 64, False, True),
                                                    (2048, 4, 40, True, False), (1024, 3, 17, False, False)])
def test_two_block_backward_matches_one_block(n, depth, rows, relu, perm, monkeypatch):
    """The two-block launch (block l+1's dx kept on chip as block l's dy) is
    bit-identical to one launch per block, for even and odd depths, with and
    without ReLU / permutations, odd row counts included."""
    from paper_1511_05946_b200 import _lib

    assert _lib.load().cascade_pair_supported(rows, n) == 1
    rng = np.random.default_rng(11)
    casc, layers, _ = build(n, depth, rng, relu=relu, perm=perm)
    x = torch.as_tensor(f32(rng, rows, n), device=DEV)
    dy = torch.as_tensor(f32(rng, rows, n), device=DEV)
    acdc = [L for L in layers if hasattr(L, "grad_a")]
    res = []
    for pair in ("1", "0"):
        monkeypatch.setenv("ACDC_CASCADE_PAIR", pair)
        casc.zero_grads()
        casc.forward(x)
        dx = casc.backward(dy)
        torch.cuda.synchronize()
        res.append([dx.clone()] + [g.clone() for L in acdc for g in (L.grad_a, L.grad_d, L.grad_bias_d)])
    for a_, b_ in zip(*res):
        assert torch.equal(a_, b_)


def test_two_block_abi_guards():
    from paper_1511_05946_b200 import _lib

    lib = _lib.load()
    assert lib.cascade_pair_supported(64, 256) == 0  # below the TMEM backward's sizes
    assert lib.cascade_pair_supported(64, 16384) == 0
    assert lib.cascade_pair_supported(0, 1024) == 0
    assert lib.cascade_pair_supported(64, 4096) == 0  # the two blocks' stashes do not fit
    assert lib.cascade_bwd_pair_defer_f32(*([None] * 12), 0, 0, None, None, 0, 64, 256, 256, 256, 256, 256,
                                          None) != 0


@pytest.mark.parametrize("n,depth,rows", [(4096, 3, 17), (4096, 12, 40), (4096, 2, 5), (4096, 1, 3), (8192, 3, 9),
                                          (16384, 2, 4), (4096, 4, 601)])
def test_hl_cascade_vs_oracle_and_paths(n, depth, rows):
    """ACDC-only stacks (the reference's acdc_cascade) at the half-length plan's
    sizes: the fused cascade (cascade_fwd_hl_f32 + deferred block backwards)
    against the fp64 oracle, and bit-identical to the per-block reductions
    (hook path) and to the per-layer (unfused) AcdcLayer path."""
    from paper_1511_05946_b200 import functional as F

    rng = np.random.default_rng(n + depth)
    casc, layers, specs = build(n, depth, rng, relu=False, perm=False, std=0.1)
    assert casc._fused is not None and casc._fused["hl"] and F.cascade_hl_supported(n)
    x = f32(rng, rows, n)
    dy = f32(rng, rows, n)
    xt, dyt = torch.as_tensor(x, device=DEV), torch.as_tensor(dy, device=DEV)
    acdc = [L for L in layers if hasattr(L, "grad_a")]
    res = []
    for mode in ("deferred", "hook", "unfused"):
        casc.zero_grads()
        fused = casc._fused
        if mode == "unfused":
            casc._fused = None
        y = casc.forward(xt)
        dx = casc.backward(dyt, on_layer=(lambda layer: None) if mode == "hook" else None)
        casc._fused = fused
        torch.cuda.synchronize()
        res.append([y.clone(), dx.clone()] + [g.clone() for L in acdc for g in (L.grad_a, L.grad_d, L.grad_bias_d)])
    for a_, b_, c_ in zip(*res):
        assert torch.equal(a_, b_)
        assert torch.equal(a_, c_)
    yr, caches = O.cascade_forward(x.astype(np.float64), specs)
    dxr, grads = O.cascade_backward(dy.astype(np.float64), specs, caches)
    grads = [g for g in grads if g is not None]
    gains = [1.0] * depth
    close(res[0][0], yr, O.chain_factor(gains) * O.fp32_tolerance(n, yr) * 2, "y")
    close(res[0][1], dxr, O.chain_factor(gains) * O.fp32_tolerance(n, dxr) * 2, "dx")
    for l, L in enumerate(acdc):
        for k, (mine, ref) in enumerate(zip((L.grad_a, L.grad_d, L.grad_bias_d), grads[l])):
            close(mine, ref, depth * O.grad_tolerance(n, rows, ref) * 2, f"block {l} grad {k}")
