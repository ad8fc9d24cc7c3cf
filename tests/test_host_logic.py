"""Host-side logic that needs no GPU: the HostPipeline chunk plan."""

import pytest

from paper_1511_05946_b200.functional import HostPipeline


@pytest.mark.parametrize("rows", [1, 2, 5, 63, 64, 100, 1000, 16384, 16385])
@pytest.mark.parametrize("chunks", [1, 3, 8, 16, 64])
@pytest.mark.parametrize("ramp", [False, True])
def test_chunk_plan_partitions_rows(rows, chunks, ramp):
    spans = HostPipeline.plan(rows, chunks, ramp)
    assert spans[0][0] == 0 and spans[-1][1] == rows
    assert all(hi > lo for lo, hi in spans)
    assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))
    assert all(lo % 2 == 0 for lo, _ in spans)  # row pairs never split across chunks
    assert len(spans) <= max(chunks, 1) + 6


def test_chunk_plan_ramp_shrinks_ends():
    sizes = [hi - lo for lo, hi in HostPipeline.plan(16384, 16, True)]
    assert sizes[0] < sizes[1] < sizes[2] < sizes[3]
    assert sizes[-1] < sizes[-2] < sizes[-3] < sizes[-4]


def test_kernel_plugin_matches_reference_signatures():
    """kernels_b200 exposes the kernel-module interface get_kernels returns
    (backend.py:30-42): COMPILED and the _kernels.pyx:49-91 signatures."""
    import inspect

    from paper_1511_05946_b200 import kernels_b200 as K

    assert K.COMPILED is True
    sig = {name: list(inspect.signature(getattr(K, name)).parameters) for name in K.__all__ if name != "COMPILED"}
    assert sig == {
        "fft_inplace": ["z", "rev", "tw", "inverse"],
        "dct2_batch": ["x", "out", "reorder", "rev", "tw", "w4s"],
        "dct3_batch": ["y", "out", "reorder", "rev", "tw", "u1", "u2"],
    }


def test_load_cascade_rejects_other_format_versions(tmp_path):
    """layers.py:548-553: the version check runs before any layer is built."""
    import json

    from paper_1511_05946_b200 import load_cascade

    p = tmp_path / "v2.json"
    p.write_text(json.dumps({"format_version": 2, "seed": None, "layers": []}))
    with pytest.raises(ValueError, match="unsupported cascade format version 2"):
        load_cascade(p)


def test_reference_cascade_files_are_format_1():
    import json
    import os

    here = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    tags = set()
    for name in ("cascade_real.json", "cascade_complex.json"):
        doc = json.load(open(os.path.join(here, name)))
        assert doc["format_version"] == 1
        tags |= {s["type"] for s in doc["layers"]}
    assert tags == {"acdc", "afdf", "relu", "permutation", "dense"}
