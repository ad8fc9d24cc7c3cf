"""CPU tier: transform plans and backend selection mirror the reference
(transforms.py:43-122, backend.py:30-42), checked against the fp64 oracle
restatement (itself pinned to the reference's golden vectors)."""

import numpy as np
import pytest

from oracle import acdc_oracle as O
from paper_1511_05946_b200.plans import DctPlan, FftPlan, dct_matrix, resolve_backend


@pytest.mark.parametrize("n", [1, 2, 8, 256, 4096])
def test_fast_plan_tables_match_oracle(n):
    p = DctPlan(n)
    t = O.tables(n)
    assert p.backend == "b200" and p.mode == "fast"
    assert np.array_equal(p.bitrev, t.rev) and np.array_equal(p.reorder, t.reorder)
    for name, ref in (("twiddle", t.tw), ("w4s", t.w4s), ("u1", t.u1), ("u2", t.u2)):
        assert np.allclose(getattr(p, name), ref, rtol=0, atol=1e-12), name


def test_naive_plan_and_errors():
    p = DctPlan(100, mode="naive")
    assert p.backend == "naive"
    assert np.allclose(p.cos_matrix, O.dct_matrix(100), atol=1e-14)
    assert np.allclose(dct_matrix(7) @ dct_matrix(7).T, np.eye(7), atol=1e-12)
    with pytest.raises(ValueError, match="power-of-two"):
        DctPlan(100)
    with pytest.raises(ValueError, match="unknown DCT mode"):
        DctPlan(8, mode="slow")
    with pytest.raises(ValueError, match="positive"):
        DctPlan(0, mode="naive")
    with pytest.raises(ValueError, match="power of two"):
        FftPlan(12)
    f = FftPlan(16)
    assert np.array_equal(f.bitrev, O.bit_reversal(16))


def test_backend_names(monkeypatch):
    for b in ("auto", "compiled", "python", "b200"):
        assert resolve_backend(b) == "b200"
    with pytest.raises(ValueError, match="unknown kernel backend"):
        resolve_backend("cuda")
    monkeypatch.setenv("ACDC_KERNEL_BACKEND", "bogus")
    with pytest.raises(ValueError, match="unknown kernel backend"):
        resolve_backend("auto")
    monkeypatch.setenv("ACDC_KERNEL_BACKEND", "python")
    assert resolve_backend("auto") == "b200"
