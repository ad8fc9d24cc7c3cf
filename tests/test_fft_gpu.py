"""GPU parity of the row FFT (acdc_fft_c64) and of the kernel-plugin module
(kernels_b200: the reference's get_kernels interface) against the oracle and
the reference's golden vectors."""

import math

import numpy as np
import pytest
import torch

from oracle import acdc_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda"


def c64(rng, *shape):
    z = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    return z.astype(np.complex64).astype(np.complex128)


def tol(n, ref):
    # SURVEY §8(c) fp32 bound, scaled by log2 N (forward DFT grows by sqrt(N): use rms of the reference)
    return O.fp32_tolerance(n, ref)


@pytest.mark.parametrize("n", [2 ** k for k in range(0, 16)])
def test_fft_ifft_match_oracle(n):
    from paper_1511_05946_b200 import functional as F

    rows = 5 if n <= 4096 else 3
    z = c64(np.random.default_rng(n), rows, n)
    zd = torch.as_tensor(z.astype(np.complex64), device=DEV)
    ref_f, ref_i = O.fft_rows(z), O.ifft_rows(z)
    got_f = F.fft(zd).cpu().numpy().astype(np.complex128)
    got_i = F.ifft(zd).cpu().numpy().astype(np.complex128)
    assert np.max(np.abs(got_f - ref_f)) <= tol(n, ref_f)
    assert np.max(np.abs(got_i - ref_i)) <= tol(n, ref_i)


def test_fft_golden_and_roundtrip(golden):
    from paper_1511_05946_b200 import functional as F

    for n in sorted({int(k.split("_")[1][1:]) for k in golden.files if k.startswith("fft_N")}):
        z = golden[f"fft_N{n}_z"]
        zd = torch.as_tensor(z.astype(np.complex64), device=DEV)
        f = F.fft(zd)
        ref = golden[f"fft_N{n}_fft"]
        assert np.max(np.abs(f.cpu().numpy() - ref)) <= tol(n, ref)
        ref = golden[f"fft_N{n}_ifft"]
        assert np.max(np.abs(F.ifft(zd).cpu().numpy() - ref)) <= tol(n, ref)
        back = F.ifft(f).cpu().numpy()
        assert np.max(np.abs(back - z)) <= tol(n, z)


def test_fft_in_place_strided_and_1d():
    from paper_1511_05946_b200 import functional as F

    n = 1024
    z = c64(np.random.default_rng(3), 7, n)
    zd = torch.as_tensor(z.astype(np.complex64), device=DEV)
    ref = F.fft(zd).clone()
    F._fft_rows(zd, False, out=zd)  # in place
    torch.testing.assert_close(zd, ref, rtol=0, atol=0)
    big = torch.zeros(7, n + 64, dtype=torch.complex64, device=DEV)
    big[:, :n] = torch.as_tensor(z.astype(np.complex64), device=DEV)
    torch.testing.assert_close(F.fft(big[:, :n]), ref, rtol=0, atol=0)
    torch.testing.assert_close(F.fft(big[2, :n]), ref[2], rtol=0, atol=0)


def test_fft_errors():
    from paper_1511_05946_b200 import functional as F

    with pytest.raises(ValueError, match="FFT size must be a power of two, got 12"):
        F.fft(torch.zeros(2, 12, dtype=torch.complex64, device=DEV))
    with pytest.raises(ValueError):
        F.fft(torch.zeros(2, 65536, dtype=torch.complex64, device=DEV))


def test_kernel_plugin_against_reference_contract(golden):
    """kernels_b200.{fft_inplace, dct2_batch, dct3_batch} on host fp64 arrays with
    the reference's plan tables, in place / into caller-owned outputs."""
    from paper_1511_05946_b200 import kernels_b200 as K

    for n in (8, 256, 1024):
        t = O.MakhoulTables(n)
        x = golden[f"dct_N{n}_x"]
        out = np.empty_like(x)
        K.dct2_batch(x, out, t.reorder, t.rev, t.tw, t.w4s)
        assert np.max(np.abs(out - golden[f"dct_N{n}_dct"])) <= O.fp32_tolerance(n, golden[f"dct_N{n}_dct"])
        K.dct3_batch(x, out, t.reorder, t.rev, t.tw, t.u1, t.u2)
        assert np.max(np.abs(out - golden[f"dct_N{n}_idct"])) <= O.fp32_tolerance(n, golden[f"dct_N{n}_idct"])
        z = golden[f"fft_N{n}_z"].copy()
        K.fft_inplace(z, t.rev, t.tw, False)
        assert np.max(np.abs(z - golden[f"fft_N{n}_fft"])) <= O.fp32_tolerance(n, golden[f"fft_N{n}_fft"])
        z = golden[f"fft_N{n}_z"].copy()
        K.fft_inplace(z, t.rev, t.tw, True)
        assert np.max(np.abs(z - golden[f"fft_N{n}_ifft"])) <= O.fp32_tolerance(n, golden[f"fft_N{n}_ifft"])
    z = np.zeros((2, 0), dtype=np.complex128)
    K.fft_inplace(z, None, None, False)  # n == 0: no-op like _kernels.pyx:53-54
