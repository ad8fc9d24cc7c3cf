"""training.py mirror: the host pieces bit-exact against the reference's own
outputs (tests/golden), the device driver on the GPU."""

import numpy as np
import pytest
import torch

from paper_1511_05946_b200 import training as T


def test_rng_streams_match_reference(golden):
    c0, c1 = T.Rng(7).spawn(2)
    np.testing.assert_array_equal(c0.uniform(3, 4), golden["train_rng_uniform"])
    np.testing.assert_array_equal(c1.gaussian(2, 5, 1.0, 0.3), golden["train_rng_gauss"])
    np.testing.assert_array_equal(T.Rng(8).permutation(10), golden["train_rng_perm"])


def test_make_regression_matches_reference(golden):
    ds = T.make_regression(3, n_samples=20, n_in=4, n_out=3)
    np.testing.assert_array_equal(ds.x, golden["train_reg_x"])
    np.testing.assert_array_equal(ds.y, golden["train_reg_y"])
    np.testing.assert_array_equal(ds.w_true, golden["train_reg_w"])
    with pytest.raises(ValueError):
        T.make_regression(0, n_samples=0)


def test_host_losses_match_reference(golden):
    p, t = golden["train_mse_in"]
    loss, grad = T.mse_loss(p, t)
    assert loss == float(golden["train_mse_loss"])
    np.testing.assert_array_equal(grad, golden["train_mse_grad"])
    loss, grad = T.softmax_cross_entropy(p, golden["train_ce_labels"])
    assert loss == float(golden["train_ce_loss"])
    np.testing.assert_array_equal(grad, golden["train_ce_grad"])


def test_init_scheme_validation():
    with pytest.raises(ValueError, match="unknown init kind"):
        T.InitScheme(kind="xavier")
    with pytest.raises(ValueError, match="sigma must be nonnegative"):
        T.InitScheme(sigma=-1.0)


@pytest.mark.gpu
def test_device_losses_match_reference(golden):
    p, t = golden["train_mse_in"]
    pd, td = torch.as_tensor(p, device="cuda"), torch.as_tensor(t, device="cuda")
    loss, grad = T.mse_loss(pd, td)
    assert loss.is_cuda and abs(float(loss) - float(golden["train_mse_loss"])) <= 1e-12
    np.testing.assert_allclose(grad.cpu().numpy(), golden["train_mse_grad"], rtol=0, atol=1e-15)
    loss, grad = T.softmax_cross_entropy(pd, torch.as_tensor(golden["train_ce_labels"], device="cuda"))
    assert abs(float(loss) - float(golden["train_ce_loss"])) <= 1e-12
    np.testing.assert_allclose(grad.cpu().numpy(), golden["train_ce_grad"], rtol=0, atol=1e-15)
    z = torch.randn(3, 4, dtype=torch.complex64, device="cuda")
    loss, grad = T.complex_mse_loss(z, torch.zeros_like(z))
    ref = np.mean(np.abs(z.cpu().numpy().astype(np.complex128)) ** 2)
    assert abs(float(loss) - ref) <= 1e-6 * ref


@pytest.mark.gpu
def test_train_curve_matches_reference(golden):
    """Same seeds / init / shuffles / schedule as the reference train(): fp32 GPU
    curve and final parameters within fp32 drift of the fp64 reference."""
    from paper_1511_05946_b200 import acdc_cascade

    ds = T.make_regression(11, n_samples=256, n_in=64, n_out=64)
    casc = acdc_cascade(64, 2)
    cfg = T.SgdConfig(learning_rate=0.002, momentum=0.9, lr_decay_factor=0.5, lr_decay_every=12)
    curve = T.train(casc, ds, cfg, init_scheme=T.InitScheme(), epochs=4, batch_size=48, seed=1)
    np.testing.assert_allclose(curve, golden["train_curve"], rtol=2e-4)
    got = np.stack([torch.cat([L.a, L.d, L.bias_d]).cpu().numpy() for L in casc.layers])
    np.testing.assert_allclose(got, golden["train_curve_params"], rtol=0, atol=2e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("check_every", [None, 1, 5])
def test_train_divergence_step_matches_reference(golden, check_every):
    from paper_1511_05946_b200 import acdc_cascade

    ds = T.make_regression(11, n_samples=256, n_in=64, n_out=64)
    bad_y = ds.y.copy()
    bad_y[200, 5] = np.nan
    casc = acdc_cascade(64, 2)
    with pytest.raises(T.DivergenceError) as e:
        T.train(casc, (ds.x, bad_y), T.SgdConfig(learning_rate=0.002, momentum=0.9), init_scheme=T.InitScheme(),
                epochs=3, batch_size=32, seed=2, check_every=check_every)
    assert int(golden["train_diverge_step"]) >= 0
    assert e.value.step == int(golden["train_diverge_step"])
