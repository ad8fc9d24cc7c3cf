"""K6: tensor-core four-step DFT vs the butterfly engine.

The DCT of one row pair is one N-point complex FFT (dct_pair.cuh).  The
four-step factorisation N = 64 x 64 turns each half of it into a batched
dense DFT-64, i.e. a GEMM: the batch of 8192 row pairs at N = 4096 becomes
[8192*64, 128] x [128, 128] (real form of the complex 64x64 DFT matrix),
17.2 GFLOP per stage, two stages per FFT (plus a twiddle pass and a
transpose, not timed here: this is a LOWER bound on the tensor-core FFT).

What is measured on one B200 (CUDA events, median of 20 after warm-up):
  * butterfly: fft_rows_kernel<12> (acdc_fft_c64), 8192 complex rows of 4096
    -- the whole FFT, in and out of HBM;
  * one four-step stage through cuBLAS (tcgen05 kernels on sm_100): TF32
    single pass, 3xTF32 (hi*hi + hi*lo + lo*hi: the fp32-accurate split),
    bf16 single pass and bf16x3;
  * the stage's error against fp64, in units of the parity bound
    4 log2(N) eps32 rms -- TF32 / bf16 single passes miss it.
cuBLAS at these shapes is the best available tensor-core GEMM and bounds
what a hand-written tcgen05 stage could do; the decision compares the
tensor-core time for the two stages with the butterfly time for the whole
FFT.  Prints one JSON line.
"""

import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import functional as F  # noqa: E402

dev = torch.device("cuda", 0)
N, R, B = 4096, 64, 8192  # row length, DFT radix per stage, row pairs (= complex rows)


NCU = os.environ.get("K6_NCU") == "1"  # one launch of each variant (for an ncu capture), no timing loops


def timed(fn, reps=20, warm=3):
    if NCU:
        fn()
        torch.cuda.synchronize()
        return float("nan")
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def tf32_hi(x):
    return (x.view(torch.int32) & -8192).view(torch.float32)  # keep 10 mantissa bits (TF32 operand)


def main():
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    z = torch.complex(torch.randn(B, N, device=dev, generator=g), torch.randn(B, N, device=dev, generator=g))
    out = torch.empty_like(z)
    F.prepare(N, dev)
    ms_fft = timed(lambda: F._fft_rows(z, False, out=out))

    # real form of the complex DFT-64: [re, im] interleaved row vector times W (128 x 128)
    k = torch.arange(R, device=dev, dtype=torch.float64)
    ang = -2 * math.pi * torch.outer(k, k) / R
    c, s = torch.cos(ang), torch.sin(ang)
    W64 = torch.zeros(2 * R, 2 * R, dtype=torch.float64, device=dev)
    W64[0::2, 0::2] = c  # out_re += in_re * cos
    W64[1::2, 0::2] = -s  # out_re -= in_im * sin
    W64[0::2, 1::2] = s  # out_im += in_re * sin
    W64[1::2, 1::2] = c  # out_im += in_im * cos
    X = torch.view_as_real(z).reshape(B * (N // R), 2 * R)  # each 64-point sub-row as 128 reals
    W = W64.float()
    res = {"n": N, "row_pairs": B, "butterfly_fft_ms": ms_fft,
           "gemm_shape": [B * (N // R), 2 * R, 2 * R], "gflop_per_stage": 2 * X.shape[0] * (2 * R) ** 2 / 1e9}
    # accuracy reference on a slice (fp64)
    sl = slice(0, 65536)
    ref = (X[sl].double() @ W64)
    rms = float(ref.pow(2).mean().sqrt())
    bound = 4 * math.log2(N) * 2.0 ** -23 * max(rms, 1.0)

    def err(y):
        return float((y[sl].double() - ref).abs().max()) / bound

    Xh, Wh = tf32_hi(X), tf32_hi(W)
    Xl, Wl = X - Xh, W - Wh
    Xb, Wb = X.bfloat16(), W.bfloat16()
    Xbl, Wbl = (X - Xb.float()).bfloat16(), (W - Wb.float()).bfloat16()
    torch.backends.cuda.matmul.allow_tf32 = True
    variants = {
        "tf32_1pass": lambda: X @ W,
        "tf32_x3": lambda: torch.addmm(torch.addmm(Xh @ Wh, Xh, Wl), Xl, Wh),
        "bf16_1pass": lambda: torch.mm(Xb, Wb, out_dtype=torch.float32),
        "bf16_x3": lambda: torch.mm(Xb, Wb, out_dtype=torch.float32) + torch.mm(Xb, Wbl, out_dtype=torch.float32)
        + torch.mm(Xbl, Wb, out_dtype=torch.float32),
    }
    for name, fn in variants.items():
        ms = timed(fn)
        y = fn()
        res[name] = {"stage_ms": ms, "two_stage_ms": 2 * ms, "vs_butterfly_fft": 2 * ms / ms_fft,
                     "err_over_parity_bound": err(y), "tflops": res["gflop_per_stage"] * (3 if "x3" in name else 1)
                     / ms}
    torch.backends.cuda.matmul.allow_tf32 = False
    res["fp32_cuda_core_gemm_stage_ms"] = timed(lambda: X @ W)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
