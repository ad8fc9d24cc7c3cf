"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (``/root/reference`` does not exist on the
GPU box):  ``python tests/golden/make_golden.py``.  Writes
``tests/golden/golden.npz``.

The reference package (``/root/reference/pkg/src/acdc``) is imported in place
(read-only).  Its compiled Cython backend is the one ``oracle/build_ref.py``
builds from the reference's own ``_kernels.pyx``; it is injected as
``acdc._kernels`` so ``backend.get_kernels("compiled")`` resolves to it
(``backend.py:20-25,38-41``).  Every input is fp32-representable (drawn in fp32,
then up-cast) so the same inputs feed the fp32 CUDA kernels in the GPU tests.

Cases (keys prefixed per case):
  dct_N*:   dct / idct of a (3, N) batch, N in {1,2,4,...,1024}   (transforms.py:137-156)
  fft_N*:   fft / ifft of a (3, N) complex batch, N in {1,...,4096} (transforms.py:166-179)
  train_*:  Rng streams, make_regression, losses, a 4-epoch training curve, a divergence step
  json_*:   reference save_cascade files cascade_{real,complex}.json (layers.py:536-554)
            and the reference forward of a batch through each
  acdc_*:   AcdcLayer forward, backward twice (accumulation)        (layers.py:141-156)
  afdf_*:   AfdfLayer forward/backward, complex                     (layers.py:199-215)
  casc_*:   Cascade of ACDC / ReLU / Permutation                    (layers.py:336-344)
  ka_*:     SPEC known answers (ones vector, identity layer, a = 0)
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
REF_SRC = "/root/reference/pkg/src"


def import_reference():
    from oracle import ref_kernels

    mod = ref_kernels.load()
    if mod is None:
        raise SystemExit("oracle/_ref could not be built")
    sys.modules["acdc._kernels"] = mod
    sys.path.insert(0, REF_SRC)
    import acdc  # noqa: E402  (the reference package)

    assert acdc.backend.get_kernels("compiled") is mod
    return acdc


def f32(rng, *shape, mean=0.0, std=1.0):
    return (mean + std * rng.standard_normal(shape)).astype(np.float32).astype(np.float64)


def main():
    acdc = import_reference()
    rng = np.random.default_rng(20251017)
    out = {}

    for n in [1, 2, 4, 8, 16, 32, 64, 128, 256, 1024]:
        plan = acdc.DctPlan(n, mode="fast", backend="compiled")
        x = f32(rng, 3, n)
        out[f"dct_N{n}_x"] = x
        out[f"dct_N{n}_dct"] = acdc.dct(plan, x)
        out[f"dct_N{n}_idct"] = acdc.idct(plan, x)

    acdc_cases = [(2, 1), (4, 3), (8, 1), (16, 3), (32, 5), (64, 2), (128, 7), (256, 4), (1024, 3)]
    for n, b in acdc_cases:
        layer = acdc.AcdcLayer(n, dct_mode="fast", backend="compiled")
        layer.a[:] = f32(rng, n, mean=1.0, std=0.4)   # gradcheck.py:98-100
        layer.d[:] = f32(rng, n, mean=1.0, std=0.4)
        layer.bias_d[:] = f32(rng, n, std=0.3)
        x = f32(rng, b, n)
        dy = f32(rng, b, n)
        y = layer.forward(x)
        dx = layer.backward(dy, retain_cache=True)
        g1 = (layer.grad_a.copy(), layer.grad_d.copy(), layer.grad_bias_d.copy())
        layer.backward(dy)  # accumulates (layers.py:152-155)
        p = f"acdc_N{n}_B{b}_"
        out[p + "a"], out[p + "d"], out[p + "bias"] = layer.a.copy(), layer.d.copy(), layer.bias_d.copy()
        out[p + "x"], out[p + "dy"], out[p + "y"], out[p + "dx"] = x, dy, y, dx
        out[p + "ga"], out[p + "gd"], out[p + "gb"] = g1
        out[p + "ga2"], out[p + "gd2"], out[p + "gb2"] = layer.grad_a.copy(), layer.grad_d.copy(), layer.grad_bias_d.copy()

    for n, b in [(4, 1), (16, 3), (64, 2), (256, 3), (1024, 2)]:
        layer = acdc.AfdfLayer(n, backend="compiled")
        layer.a[:] = f32(rng, n, mean=1.0, std=0.3) + 1j * f32(rng, n, std=0.3)  # gradcheck.py:105-106
        layer.d[:] = f32(rng, n, mean=1.0, std=0.3) + 1j * f32(rng, n, std=0.3)
        x = f32(rng, b, n) + 1j * f32(rng, b, n)
        dy = f32(rng, b, n) + 1j * f32(rng, b, n)
        y = layer.forward(x)
        dx = layer.backward(dy)
        p = f"afdf_N{n}_B{b}_"
        out[p + "a"], out[p + "d"], out[p + "x"], out[p + "dy"] = layer.a.copy(), layer.d.copy(), x, dy
        out[p + "y"], out[p + "dx"], out[p + "ga"], out[p + "gd"] = y, dx, layer.grad_a.copy(), layer.grad_d.copy()

    # cascade: ACDC -> ReLU -> Perm repeated, no ReLU/Perm after the last ACDC
    for n, depth, b in [(16, 3, 4), (64, 4, 3), (256, 3, 2)]:
        prng = acdc.Rng(7 + n)
        layers = []
        for i in range(depth):
            L = acdc.AcdcLayer(n, backend="compiled")
            L.a[:] = f32(rng, n, mean=1.0, std=0.2)
            L.d[:] = f32(rng, n, mean=1.0, std=0.2)
            L.bias_d[:] = f32(rng, n, std=0.1)
            layers.append(L)
            if i < depth - 1:
                layers.append(acdc.ReluLayer(n))
                layers.append(acdc.PermutationLayer(n, rng=prng))
        cas = acdc.Cascade(layers)
        x = f32(rng, b, n)
        dy = f32(rng, b, n)
        y = cas.forward(x)
        dx = cas.backward(dy)
        p = f"casc_N{n}_K{depth}_B{b}_"
        out[p + "x"], out[p + "dy"], out[p + "y"], out[p + "dx"] = x, dy, y, dx
        li = 0
        for L in layers:
            if isinstance(L, acdc.AcdcLayer):
                for nm in ("a", "d", "bias_d", "grad_a", "grad_d", "grad_bias_d"):
                    out[p + f"L{li}_{nm}"] = getattr(L, nm).copy()
                li += 1
            elif isinstance(L, acdc.PermutationLayer):
                out[p + f"P{li - 1}_perm"] = L.perm.copy()

    # SPEC known answers
    n = 16
    plan = acdc.DctPlan(n, backend="compiled")
    out["ka_dct_ones16"] = acdc.dct(plan, np.ones((1, n)))
    ident = acdc.AcdcLayer(n, backend="compiled")
    x = f32(rng, 2, n)
    out["ka_ident_x"], out["ka_ident_y"] = x, ident.forward(x)
    out["ka_ident_dx"] = ident.backward(x)
    z = acdc.AcdcLayer(n, backend="compiled")
    z.a[:] = 0.0
    z.bias_d[:] = f32(rng, n)
    out["ka_a0_bias"], out["ka_a0_y"] = z.bias_d.copy(), z.forward(x)

    # fft_N*: fft / ifft of a (3, N) complex batch (transforms.py:166-179);
    # own generator so the arrays above keep their values
    frng = np.random.default_rng(20261017)
    for n in [1, 2, 4, 8, 16, 32, 64, 128, 256, 1024, 4096]:
        plan = acdc.FftPlan(n, backend="compiled")
        z = f32(frng, 3, n) + 1j * f32(frng, 3, n)
        out[f"fft_N{n}_z"] = z
        out[f"fft_N{n}_fft"] = acdc.fft(plan, z)
        out[f"fft_N{n}_ifft"] = acdc.ifft(plan, z)

    # json_*: cascades written by the reference's save_cascade (layers.py:536-545)
    # with fp32-representable parameters, plus the reference forward of a batch
    here = os.path.dirname(os.path.abspath(__file__))
    jrng = np.random.default_rng(20261018)
    n = 16
    l0 = acdc.AcdcLayer(n)
    l3 = acdc.AcdcLayer(n)
    for L in (l0, l3):
        L.a[:] = f32(jrng, n, mean=1.0, std=0.3)
        L.d[:] = f32(jrng, n, mean=1.0, std=0.3)
        L.bias_d[:] = f32(jrng, n, std=0.2)
    dense = acdc.DenseLayer(n, 8)
    dense.w[...] = f32(jrng, n, 8, std=0.3)
    dense.b[:] = f32(jrng, 8, std=0.1)
    real = acdc.Cascade([l0, acdc.ReluLayer(n), acdc.PermutationLayer(n, rng=acdc.Rng(5)), l3, dense])
    acdc.save_cascade(real, os.path.join(here, "cascade_real.json"), seed=5)
    x = f32(jrng, 4, n)
    out["json_real_x"], out["json_real_y"] = x, real.forward(x)
    f0 = acdc.AfdfLayer(n, fix_a=True)
    f2 = acdc.AfdfLayer(n)
    for L in (f0, f2):
        L.a[:] = f32(jrng, n, mean=1.0, std=0.2) + 1j * f32(jrng, n, std=0.2)
        L.d[:] = f32(jrng, n, mean=1.0, std=0.2) + 1j * f32(jrng, n, std=0.2)
    cplx = acdc.Cascade([f0, acdc.PermutationLayer(n, rng=acdc.Rng(6)), f2])
    acdc.save_cascade(cplx, os.path.join(here, "cascade_complex.json"))
    z = f32(jrng, 4, n) + 1j * f32(jrng, 4, n)
    out["json_cplx_x"], out["json_cplx_y"] = z, cplx.forward(z)

    # train_*: training.py pieces — Rng streams, make_regression, host losses,
    # a short reference training curve and a divergence step
    r = acdc.Rng(7)
    c0, c1 = r.spawn(2)
    out["train_rng_uniform"] = c0.uniform(3, 4)
    out["train_rng_gauss"] = c1.gaussian(2, 5, 1.0, 0.3)
    out["train_rng_perm"] = acdc.Rng(8).permutation(10)
    ds = acdc.make_regression(3, n_samples=20, n_in=4, n_out=3)
    out["train_reg_x"], out["train_reg_y"], out["train_reg_w"] = ds.x, ds.y, ds.w_true
    lrng = np.random.default_rng(5)
    p_, t_ = lrng.standard_normal((4, 6)), lrng.standard_normal((4, 6))
    out["train_mse_in"] = np.stack([p_, t_])
    out["train_mse_loss"], out["train_mse_grad"] = np.float64(acdc.mse_loss(p_, t_)[0]), acdc.mse_loss(p_, t_)[1]
    labels = np.array([0, 5, 2, 3])
    out["train_ce_labels"] = labels
    out["train_ce_loss"], out["train_ce_grad"] = (np.float64(acdc.softmax_cross_entropy(p_, labels)[0]),
                                                  acdc.softmax_cross_entropy(p_, labels)[1])
    ds = acdc.make_regression(11, n_samples=256, n_in=64, n_out=64)
    casc = acdc.acdc_cascade(64, 2)
    cfg = acdc.SgdConfig(learning_rate=0.002, momentum=0.9, lr_decay_factor=0.5, lr_decay_every=12)
    out["train_curve"] = np.array(acdc.train(casc, ds, cfg, init_scheme=acdc.InitScheme(), epochs=4,
                                             batch_size=48, seed=1))
    out["train_curve_params"] = np.stack([np.concatenate([L.a, L.d, L.bias_d]) for L in casc.layers])
    casc = acdc.acdc_cascade(64, 2)
    bad_y = ds.y.copy()
    bad_y[200, 5] = np.nan  # one poisoned target: diverges at the step whose batch holds sample 200
    try:
        acdc.train(casc, (ds.x, bad_y), acdc.SgdConfig(learning_rate=0.002, momentum=0.9),
                   init_scheme=acdc.InitScheme(), epochs=3, batch_size=32, seed=2)
        out["train_diverge_step"] = np.int64(-1)
    except acdc.DivergenceError as e:
        out["train_diverge_step"] = np.int64(e.step)

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
