"""Time the 64 x 64 two-pass FFT probe (scripts/r64_probe.cu, built into
gpurun_variants/r64_*.so) against the engine's radix-16 row FFT and cuFFT on
batched N=4096 complex64 rows.  CUDA-graph replay.  Experimental probe.

  python scripts/r64_probe.py lib.so[:grid_per_sm] ...
"""

import ctypes
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_05946_b200 import functional as F  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from fft_vs_cufft import timed  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    n = 4096
    F.prepare(n, dev)
    n1 = np.arange(64)[:, None]
    m = np.arange(8)[None, :]
    ang = np.concatenate([-2 * math.pi * n1 * m / n, -2 * math.pi * 8 * n1 * m / n], axis=1)
    tw = torch.tensor(np.stack([np.cos(ang), np.sin(ang)], -1).astype(np.float32), device=dev).transpose(0, 1).contiguous()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    for spec in sys.argv[1:]:
        path, _, per = spec.partition(":")
        per = int(per or 1)
        lib = ctypes.CDLL(os.path.abspath(path))
        lib.r64_k.restype = ctypes.c_int
        lib.r64_fft.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
        gpc = lib.r64_gpc()
        for rows in (2048, 8192, 32768):
            z = torch.randn(rows, n, dtype=torch.complex64, device=dev)
            out = torch.empty_like(z)
            grid = min(sms * per, (rows + gpc - 1) // gpc)

            def run():
                rc = lib.r64_fft(z.data_ptr(), out.data_ptr(), tw.data_ptr(), rows, grid,
                                 torch.cuda.current_stream().cuda_stream)
                assert rc == 0, rc

            run()
            torch.cuda.synchronize()
            K = lib.r64_k()
            ref = z.to(torch.complex128)
            for k in range(K):
                ref = torch.fft.fft(ref) / (4096.0 if k else 1.0)
            ref = ref.to(torch.complex64)
            err = float((out - ref).abs().max() / ref.abs().max())
            eng = F._fft_rows(z, False)
            err_eng = float((eng - ref).abs().max() / ref.abs().max())
            t_r64 = timed(run)
            t_eng = timed(lambda: F._fft_rows(z, False, out=out))
            print(json.dumps({"lib": os.path.basename(path), "k": K, "grid_per_sm": per, "gpc": gpc, "rows": rows,
                              "r64_us": t_r64 * 1e3, "engine_us": t_eng * 1e3, "speedup": t_eng / t_r64,
                              "r64_rel_err": err, "engine_rel_err": err_eng}), flush=True)


if __name__ == "__main__":
    main()
