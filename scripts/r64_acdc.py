"""Check and time the radix-64 ACDC forward prototype (scripts/r64_acdc.cu)
against the library forward (recompute mode) at N=4096.  Experimental probe.

  python scripts/r64_acdc.py lib.so [rows]
"""

import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from fft_vs_cufft import timed  # noqa: E402
from paper_1511_05946_b200 import functional as F  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    n = 4096
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    F.prepare(n, dev)
    lib = ctypes.CDLL(os.path.abspath(sys.argv[1]))
    lib.r64_fwd.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    x = torch.randn(rows, n, device=dev, generator=g)
    a = 1 + 0.1 * torch.randn(n, device=dev, generator=g)
    d = 1 + 0.1 * torch.randn(n, device=dev, generator=g)
    b = 0.1 * torch.randn(n, device=dev, generator=g)
    y = torch.empty_like(x)
    y_ref = F.acdc_forward(x, a, d, b)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    gpc = lib.r64_gpc()
    for per in (1,):
        grid = min(sms * per, (rows // 2 + gpc - 1) // gpc)

        def run():
            rc = lib.r64_fwd(x.data_ptr(), y.data_ptr(), a.data_ptr(), d.data_ptr(), b.data_ptr(), rows, grid,
                             torch.cuda.current_stream().cuda_stream)
            assert rc == 0, rc

        run()
        torch.cuda.synchronize()
        err = float((y - y_ref).abs().max())
        rms = float(y_ref.pow(2).mean().sqrt())
        t_r64 = timed(run)
        t_lib = timed(lambda: F.acdc_forward(x, a, d, b, out=y_ref))
        print(json.dumps({"rows": rows, "grid": grid, "gpc": gpc, "r64_us": t_r64 * 1e3, "lib_recompute_us": t_lib * 1e3,
                          "speedup": t_lib / t_r64, "max_abs_err_vs_lib": err, "rms": rms,
                          "tol_4log2N_eps": 4 * 12 * 1.1920929e-07 * max(rms, 1.0)}), flush=True)


if __name__ == "__main__":
    main()
