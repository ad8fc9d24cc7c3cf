"""Build recipe for ``oracle/_ref`` — the reference's own compiled CPU kernels.

TEST / BASELINE INFRASTRUCTURE.  Compiles the reference's single native
module, ``/root/reference/pkg/src/acdc/_kernels.pyx`` (Cython -> C, ``-O3``,
the same flags as the reference ``setup.py:11-17``), from the source where it
lies.  Outputs go only to ``oracle/_ref/`` (git-ignored; it still travels to
the GPU box with ``gpurun`` so ``bench.py --impl reference`` can time it).
No reference source is copied into the repository: the generated C file and
the shared object are build products.

Usage: ``python oracle/build_ref.py`` (no-op when the .so is newer than the
.pyx, or when ``/root/reference`` is absent, e.g. on the GPU box).
"""

from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
PYX = "/root/reference/pkg/src/acdc/_kernels.pyx"
EXT = sysconfig.get_config_var("EXT_SUFFIX") or ".so"
SO = os.path.join(OUT, "_kernels" + EXT)


def build(verbose: bool = False) -> str | None:
    if not os.path.exists(PYX):
        return SO if os.path.exists(SO) else None
    if os.path.exists(SO) and os.path.getmtime(SO) >= os.path.getmtime(PYX):
        return SO
    import numpy as np

    os.makedirs(OUT, exist_ok=True)
    c_file = os.path.join(OUT, "_kernels.c")
    # module name "acdc._kernels" is what the reference builds (setup.py:11-12)
    subprocess.run(
        [sys.executable, "-m", "cython", "-3", "--module-name", "acdc._kernels", PYX, "-o", c_file],
        check=True,
        capture_output=not verbose,
    )
    inc_py = sysconfig.get_paths()["include"]
    cmd = [
        "gcc", "-O3", "-shared", "-fPIC", "-pthread",
        "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION",
        f"-I{inc_py}", f"-I{np.get_include()}",
        c_file, "-o", SO,
    ]
    subprocess.run(cmd, check=True, capture_output=not verbose)
    os.remove(c_file)  # keep only the build product in oracle/_ref
    return SO


if __name__ == "__main__":
    path = build(verbose=True)
    print(path or "reference source absent and no prebuilt _ref")
