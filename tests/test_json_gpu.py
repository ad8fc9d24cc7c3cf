"""Cascade JSON interop (layers.py:466-554): files written by the reference's
save_cascade load into GPU layers, reproduce the reference forward, and save
back to the same document."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import acdc_oracle as O

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("name,key", [("cascade_real.json", "json_real"), ("cascade_complex.json", "json_cplx")])
def test_reference_file_loads_runs_and_saves_back(tmp_path, golden, name, key):
    from paper_1511_05946_b200 import load_cascade, save_cascade

    src = os.path.join(HERE, name)
    casc = load_cascade(src)
    x, ref = golden[key + "_x"], golden[key + "_y"]
    y = casc.forward(x)  # host array in -> float64 / complex128 numpy out, like the reference
    assert isinstance(y, np.ndarray) and y.shape == ref.shape
    assert np.max(np.abs(y - ref)) <= O.fp32_tolerance(16, ref) * 4
    out = tmp_path / "back.json"
    save_cascade(casc, out, seed=json.load(open(src))["seed"])
    assert json.load(open(out)) == json.load(open(src))  # fp32-representable values: exact


def test_save_load_roundtrip_bit_exact(tmp_path):
    from paper_1511_05946_b200 import AcdcLayer, AfdfLayer, Cascade, PermutationLayer, ReluLayer, load_cascade, save_cascade

    n = 256
    rng = np.random.default_rng(0)
    layers = []
    for i in range(3):
        L = AcdcLayer(n)
        L.a.normal_(1.0, 0.1), L.d.normal_(1.0, 0.1), L.bias_d.normal_(0.0, 0.1)
        layers += [L, ReluLayer(n), PermutationLayer(n, rng=rng)]
    casc = Cascade(layers[:-2])
    p = tmp_path / "c.json"
    save_cascade(casc, p)
    back = load_cascade(p)
    for u, v in zip(casc.params(), back.params()):
        assert torch.equal(u.value, v.value)
    x = torch.randn(64, n, device="cuda")
    torch.testing.assert_close(back.forward(x), casc.forward(x), rtol=0, atol=0)
    f = Cascade([AfdfLayer(64, fix_a=True), AfdfLayer(64)])
    for L in f.layers:
        L.a.copy_(torch.randn(64, dtype=torch.complex64))
        L.d.copy_(torch.randn(64, dtype=torch.complex64))
    save_cascade(f, p)
    g = load_cascade(p)
    assert [L.fix_a for L in g.layers] == [True, False]
    for u, v in zip(f.layers, g.layers):
        assert torch.equal(u.a, v.a) and torch.equal(u.d, v.d)


def test_bad_documents(tmp_path):
    from paper_1511_05946_b200 import load_cascade

    p = tmp_path / "bad.json"
    p.write_text(json.dumps({"format_version": 1, "layers": [{"type": "conv", "n": 4}]}))
    with pytest.raises(ValueError, match="unknown layer tag 'conv'"):
        load_cascade(p)


def test_permutation_keeps_complex_dtype():
    """PermutationLayer is dtype-agnostic (layers.py:256-265): complex in, complex out."""
    from paper_1511_05946_b200 import PermutationLayer

    P = PermutationLayer(8, perm=[3, 1, 0, 2, 7, 6, 5, 4])
    z = (np.arange(16) + 1j * np.arange(16)).reshape(2, 8)
    y = P.forward(z)
    assert np.iscomplexobj(y)
    np.testing.assert_array_equal(y, z[:, P.perm])
    np.testing.assert_array_equal(P.backward(y), z)
    zt = torch.as_tensor(z, dtype=torch.complex64, device="cuda")
    assert P.forward(zt).dtype == torch.complex64
