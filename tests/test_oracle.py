"""CPU tier: pin the fp64 oracle against the reference's golden vectors and the
SPEC known answers."""

import math

import numpy as np
import pytest

from oracle import acdc_oracle as O


def _cases(golden, prefix, strip="_x"):
    """Case prefixes: keys ending in "_x", with ``strip`` removed."""
    return sorted({k[: -len(strip)] for k in golden.files if k.startswith(prefix) and k.endswith("_x")})


def test_dct_matches_reference(golden):
    cases = _cases(golden, "dct_N")
    assert len(cases) >= 10
    for p in cases:
        x = golden[p + "_x"]
        np.testing.assert_allclose(O.dct2_rows(x), golden[p + "_dct"], atol=1e-13, rtol=0)
        np.testing.assert_allclose(O.dct3_rows(x), golden[p + "_idct"], atol=1e-13, rtol=0)


def test_fft_matches_reference(golden):
    ns = sorted({int(k.split("_")[1][1:]) for k in golden.files if k.startswith("fft_N")})
    assert len(ns) >= 10
    for n in ns:
        z = golden[f"fft_N{n}_z"]
        np.testing.assert_allclose(O.fft_rows(z), golden[f"fft_N{n}_fft"], atol=1e-12, rtol=0)
        np.testing.assert_allclose(O.ifft_rows(z), golden[f"fft_N{n}_ifft"], atol=1e-13, rtol=0)


def test_dct_matches_naive_matrix():
    rng = np.random.default_rng(0)
    for n in [1, 2, 8, 64, 1024]:
        x = rng.standard_normal((3, n))
        c = O.dct_matrix(n)
        np.testing.assert_allclose(O.dct2_rows(x), x @ c, atol=1e-10)
        np.testing.assert_allclose(O.dct3_rows(x), x @ c.T, atol=1e-10)


def test_acdc_matches_reference(golden):
    cases = _cases(golden, "acdc_N", "x")
    assert len(cases) >= 9
    for p in cases:
        g = lambda k: golden[p + k]
        y, h2 = O.acdc_forward(g("x"), g("a"), g("d"), g("bias"))
        np.testing.assert_allclose(y, g("y"), atol=1e-13)
        grads = (np.zeros_like(g("a")), np.zeros_like(g("a")), np.zeros_like(g("a")))
        dx, ga, gd, gb = O.acdc_backward(g("x"), h2, g("dy"), g("a"), g("d"), grads)
        np.testing.assert_allclose(dx, g("dx"), atol=1e-13)
        for mine, ref in ((ga, "ga"), (gd, "gd"), (gb, "gb")):
            np.testing.assert_allclose(mine, g(ref), atol=1e-12)
        O.acdc_backward(g("x"), h2, g("dy"), g("a"), g("d"), grads)  # accumulate twice
        for mine, ref in zip(grads, ("ga2", "gd2", "gb2")):
            np.testing.assert_allclose(mine, g(ref), atol=1e-12)


def test_afdf_matches_reference(golden):
    for p in _cases(golden, "afdf_N", "x"):
        g = lambda k: golden[p + k]
        y, h2 = O.afdf_forward(g("x"), g("a"), g("d"))
        np.testing.assert_allclose(y, g("y"), atol=1e-13)
        dx, ga, gd = O.afdf_backward(g("x"), h2, g("dy"), g("a"), g("d"))
        np.testing.assert_allclose(dx, g("dx"), atol=1e-12)
        np.testing.assert_allclose(ga, g("ga"), atol=1e-12)
        np.testing.assert_allclose(gd, g("gd"), atol=1e-12)


def test_cascade_matches_reference(golden):
    cases = _cases(golden, "casc_N")
    assert cases
    for p in cases:
        n = int(p.split("_N")[1].split("_")[0])
        depth = int(p.split("_K")[1].split("_")[0])
        specs = []
        for i in range(depth):
            specs.append({"kind": "acdc", "a": golden[p + f"_L{i}_a"], "d": golden[p + f"_L{i}_d"],
                          "bias": golden[p + f"_L{i}_bias_d"]})
            if i < depth - 1:
                specs.append({"kind": "relu"})
                specs.append({"kind": "perm", "perm": golden[p + f"_P{i}_perm"]})
        y, caches = O.cascade_forward(golden[p + "_x"], specs)
        np.testing.assert_allclose(y, golden[p + "_y"], atol=1e-12)
        dx, grads = O.cascade_backward(golden[p + "_dy"], specs, caches)
        np.testing.assert_allclose(dx, golden[p + "_dx"], atol=1e-12)
        li = 0
        for i, s in enumerate(specs):
            if s["kind"] == "acdc":
                ga, gd, gb = grads[i]
                np.testing.assert_allclose(ga, golden[p + f"_L{li}_grad_a"], atol=1e-12)
                np.testing.assert_allclose(gd, golden[p + f"_L{li}_grad_d"], atol=1e-12)
                np.testing.assert_allclose(gb, golden[p + f"_L{li}_grad_bias_d"], atol=1e-12)
                li += 1


def test_spec_known_answers(golden):
    # dct(ones_N) = (sqrt N, 0, ...)
    out = O.dct2_rows(np.ones((1, 16)))
    np.testing.assert_allclose(out, golden["ka_dct_ones16"], atol=1e-14)
    assert abs(out[0, 0] - 4.0) < 1e-14 and np.abs(out[0, 1:]).max() < 1e-14
    # identity layer: y = x and dx = dy
    x = golden["ka_ident_x"]
    one, zero = np.ones(16), np.zeros(16)
    y, h2 = O.acdc_forward(x, one, one, zero)
    np.testing.assert_allclose(y, x, atol=1e-14)
    np.testing.assert_allclose(y, golden["ka_ident_y"], atol=1e-14)
    dx, *_ = O.acdc_backward(x, h2, x, one, one)
    np.testing.assert_allclose(dx, golden["ka_ident_dx"], atol=1e-14)
    # a = 0 => y = idct(bias)
    y0, _ = O.acdc_forward(x, zero, one, golden["ka_a0_bias"])
    np.testing.assert_allclose(y0, golden["ka_a0_y"], atol=1e-14)
    np.testing.assert_allclose(y0[0], O.dct3_rows(golden["ka_a0_bias"][None])[0], atol=1e-14)
    # dy = 0 => zero grads
    dx, ga, gd, gb = O.acdc_backward(x, h2, np.zeros_like(x), one, one)
    assert not dx.any() and not ga.any() and not gd.any() and not gb.any()
    # FFT of impulse = ones, of constant = (cN, 0, ...)
    imp = np.zeros((1, 8), complex)
    imp[0, 0] = 1
    np.testing.assert_allclose(O.fft_rows(imp), np.ones((1, 8)), atol=1e-15)
    np.testing.assert_allclose(O.fft_rows(np.full((1, 8), 2.0 + 0j))[0], [16] + [0] * 7, atol=1e-14)


def test_tolerance_functions():
    ref = np.ones((4, 4096))
    tol = O.fp32_tolerance(4096, ref)
    assert math.isclose(tol, 4 * 12 * 2**-23, rel_tol=1e-12)
    assert O.grad_tolerance(4096, 16384, np.full(4, 3.0)) > O.grad_tolerance(4096, 2, np.full(4, 3.0))


def test_roundtrip_and_orthogonality():
    rng = np.random.default_rng(1)
    for n in [64, 4096]:
        x = rng.standard_normal((2, n))
        np.testing.assert_allclose(O.dct3_rows(O.dct2_rows(x)), x, atol=1e-12)


def test_ref_kernels_agree_with_oracle():
    from oracle import ref_kernels

    if ref_kernels.load() is None:
        pytest.skip("oracle/_ref not built and reference source absent")
    rng = np.random.default_rng(2)
    n, b = 256, 9
    a, d, bias = 1 + 0.1 * rng.standard_normal((3, n))
    x, dy = rng.standard_normal((2, b, n))
    layer = ref_kernels.RefAcdc(a, d, bias)
    y, dx, ga, gd, gb = ref_kernels.fwd_bwd_threaded(layer, x, dy, threads=3)
    yo, h2 = O.acdc_forward(x, a, d, bias)
    dxo, gao, gdo, gbo = O.acdc_backward(x, h2, dy, a, d)
    for m, r in ((y, yo), (dx, dxo), (ga, gao), (gd, gdo), (gb, gbo)):
        np.testing.assert_allclose(m, r, atol=1e-12)


def test_sgd_matches_reference_update():
    """paper_1511_05946_b200.training.Sgd == training.py:72-84 (oracle.sgd_step), CPU tensors."""
    import torch

    from paper_1511_05946_b200.layers import Param
    from paper_1511_05946_b200.training import Sgd, SgdConfig

    rng = np.random.default_rng(4)
    vals = [rng.standard_normal(5) for _ in range(3)]
    grads = [rng.standard_normal(5) for _ in range(3)]
    decay = [False, True, False]
    mult = [1.0, 0.5, 2.0]
    ps = [Param(f"p{i}", torch.tensor(v), torch.tensor(g), decay=dc, lr_mult=m)
          for i, (v, g, dc, m) in enumerate(zip(vals, grads, decay, mult))]
    cfg = SgdConfig(learning_rate=0.1, momentum=0.9, weight_decay=0.01, lr_decay_factor=0.5, lr_decay_every=2)
    opt = Sgd(ps, cfg)
    ref_v = [np.zeros(5) for _ in range(3)]
    ref_p = [v.copy() for v in vals]
    for step in range(3):
        gs = [rng.standard_normal(5) for _ in range(3)]
        for p, g in zip(ps, gs):
            p.grad.copy_(torch.tensor(g))
        opt.step()
        for i in range(3):
            gg = gs[i].copy()
            O.sgd_step(ref_p[i], gg, ref_v[i], cfg.effective_lr(step), cfg.momentum, cfg.weight_decay, decay[i], mult[i])
    for p, r in zip(ps, ref_p):
        np.testing.assert_allclose(p.value.numpy(), r, atol=1e-12)
        assert float(p.grad.abs().sum()) == 0.0


def test_ref_afdf_and_chain_tolerance():
    """The reference-compiled AFDF driver (used by the full-shape GPU tests)
    agrees with the numpy restatement; chain_factor sums gain products."""
    from oracle import ref_kernels

    if ref_kernels.load() is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(3)
    n, rows = 64, 9
    c = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)
    x, dy, a, d = c(rows, n), c(rows, n), 1 + 0.1 * c(n), 1 + 0.1 * c(n)
    y, dx, ga, gd = ref_kernels.afdf_fwd_bwd_threaded(x, dy, a, d, threads=2)
    yr, h2 = O.afdf_forward(x, a, d)
    dxr, gar, gdr = O.afdf_backward(x, h2, dy, a, d)
    for m, r in ((y, yr), (dx, dxr), (ga, gar), (gd, gdr)):
        assert np.abs(m - r).max() < 1e-9 * max(1.0, np.abs(r).max())
    assert O.chain_factor([1.0] * 5) == 5.0
    assert abs(O.chain_factor([2.0, 2.0, 2.0]) - 7.0) < 1e-12  # 1 + 2 + 4
    assert abs(O.block_gain(np.ones(8), 2 * np.ones(8)) - 2.0) < 1e-12
