"""CPU tier: the C-ABI library loads and exports every symbol the header
declares; argument validation that needs no GPU."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "acdc_b200.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b((?:acdc|afdf|cascade)_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1511_05946_b200 import _lib, build

    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    return _lib.load()


def test_header_symbols_exported(lib):
    names = _declared()
    assert "acdc_fwd_f32" in names and "acdc_bwd_f32" in names
    for name in names:
        assert hasattr(lib, name), f"{name} declared in acdc_b200.h but not exported"


def test_binding_covers_header():
    from paper_1511_05946_b200 import _lib

    assert set(_declared()) == set(_lib.SIGNATURES)


def test_abi_version_and_errors(lib):
    from paper_1511_05946_b200 import _lib

    assert lib.acdc_abi_version() == _lib.ABI_VERSION
    assert lib.acdc_max_n() == 32768
    # non-power-of-two n: the reference's ValueError message (transforms.py:96-97)
    assert lib.acdc_prepare(12) == _lib.ACDC_E_SIZE
    assert b"power-of-two" in lib.acdc_strerror(_lib.ACDC_E_SIZE)
    with pytest.raises(ValueError, match="power-of-two size, got 12"):
        _lib.check(lib.acdc_prepare(12))
    assert lib.acdc_prepare(65536) == _lib.ACDC_E_SIZE
    # shape validation happens before any device work
    assert lib.acdc_fwd_f32(None, None, None, None, None, 4, 16, 8, 16, None) == _lib.ACDC_E_SHAPE
    assert lib.acdc_fwd_f32(None, None, None, None, None, -1, 16, 16, 16, None) == _lib.ACDC_E_SHAPE
    assert lib.acdc_fwd_f32(None, None, None, None, None, 4, 16, 16, 16, None) == _lib.ACDC_E_NULL
    assert lib.acdc_dct2_f32(None, None, 3, 16, 16, 16, None) == _lib.ACDC_E_NULL
    assert lib.acdc_bwd_workspace_bytes(16, 12) == 0
    for code in (-2, -3, -4, -6):
        assert lib.acdc_strerror(code)


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_1511_05946_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|\"\"\"[\s\S]*?\"\"\"", "", src), f


def test_sgd_entry_validation(lib):
    """acdc_bwd_sgd_f32 rejects a missing step descriptor and a block epilogue
    without the h2 cache before any device work."""
    from paper_1511_05946_b200 import _lib

    f = lib.acdc_bwd_sgd_f32
    assert f(None, None, None, None, None, 0, None, None, None, 0, None, None, 0, 4, 16, 16, 16, 16, None) == \
        _lib.ACDC_E_NULL
    st = _lib.SgdStep()
    for k in range(3):  # never dereferenced: validation fails first
        st.value[k] = 0x1000 + 64 * k
        st.velocity[k] = 0x2000 + 64 * k
    assert f(None, None, None, None, None, 1, None, None, None, 0, ctypes.byref(st), None, 0, 4, 256, 256, 256, 256,
             None) == _lib.ACDC_E_SHAPE
    st.velocity[1] = None
    assert f(None, None, None, None, None, 0, None, None, None, 0, ctypes.byref(st), None, 0, 4, 256, 256, 256, 256,
             None) == _lib.ACDC_E_NULL


def test_step_entry_limits(lib):
    """The fused small-batch step: sizes and row limits (host logic, no GPU)."""
    from paper_1511_05946_b200 import _lib

    assert lib.acdc_step_max_rows(128) == 0 and lib.acdc_step_max_rows(8192) == 0
    assert lib.acdc_step_max_rows(256) >= 128  # C1 (n = 256, 128 rows) is one launch
    assert lib.acdc_step_max_rows(4096) == 0  # the separate half-length kernels are faster there
    for n in (256, 512, 1024, 2048):
        assert lib.acdc_step_max_rows(n) > 0
    rc = lib.acdc_step_f32(None, None, None, None, None, None, None, None, None, None, 0, 4, 128, 128, 128, 128, 128,
                           None)
    assert rc == _lib.ACDC_E_SIZE
    big = lib.acdc_step_max_rows(256) + 1
    rc = lib.acdc_step_f32(None, None, None, None, None, None, None, None, None, None, 0, big, 256, 256, 256, 256,
                           256, None)
    assert rc == _lib.ACDC_E_SIZE
