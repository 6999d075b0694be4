"""Layer bundles: the reference's on-disk layer format read by the
product's C-ABI bundle reader (host side, no GPU needed) — round trips against the
reference's own save_layer (oracle/_ref) and the reference tests' failure KATs
(test_container.cpp:70-107, test_runtime.cpp:452-482)."""
import json
import shutil
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import REF_SO, make_layer, ref

pytestmark = pytest.mark.skipif(not REF_SO.exists(), reason="oracle/_ref not built (needs /root/reference)")


def q():
    import paper_2310_09259_b200 as m

    return m


@pytest.mark.parametrize("bits,O,bias,sparse", [(4, 16, True, False), (8, 8, False, False), (4, 0, True, False),
                                                (4, 8, True, True)])
def test_bundle_round_trip_matches_reference_save_layer(tmp_path, bits, O, bias, sparse):
    m = q()
    r = ref()
    rng = np.random.default_rng(173 + bits + O)
    L, x, w = make_layer(rng, 4, 48, 12, bits, O, heavy_cols=1, with_bias=bias, checker=r)
    mask = None
    if sparse:
        st, sq = r.sparsegpt_joint(w, np.asarray(L["idx"], np.int64), bits)
        assert st == 0
        L.update(base=sq["base"], scales=sq["scales"], wreduced=sq["wreduced"], outlier_weights=sq["outlier_weights"])
        mask = sq["mask"]
    d = tmp_path / "layer"
    assert r.save_layer(d, L, mask=mask, wfp32=w) == 0
    got = m.load_layer(d)
    assert got.act_bits == bits and got.weights.bits() == bits
    np.testing.assert_array_equal(got.weights.base.data, np.asarray(L["base"], np.uint8))
    np.testing.assert_array_equal(got.weights.scales.view(np.uint32), np.asarray(L["scales"], np.float32).view(np.uint32))
    np.testing.assert_array_equal(got.weights.wreduced.view(np.uint32),
                                  np.asarray(L["wreduced"], np.float32).view(np.uint32))
    np.testing.assert_array_equal(got.weights.outlier_weights.reshape(-1),
                                  np.asarray(L["outlier_weights"], np.float32).reshape(-1))
    np.testing.assert_array_equal(got.outliers.indices, np.asarray(L["idx"], np.int64))
    if bias:
        np.testing.assert_array_equal(got.bias, L["bias"])
    else:
        assert got.bias is None
    if sparse:
        np.testing.assert_array_equal(got.weights.mask, mask)
    else:
        assert got.weights.mask is None


def _bundle(tmp_path, name="layer"):
    r = ref()
    rng = np.random.default_rng(5)
    L, x, w = make_layer(rng, 4, 40, 8, 4, 8, heavy_cols=1, checker=r)
    d = tmp_path / name
    assert r.save_layer(d, L) == 0
    return d


def _patch(d, fn):
    mf = d / "manifest.json"
    j = json.loads(mf.read_text())
    fn(j)
    mf.write_text(json.dumps(j, indent=2))


def test_bundle_failure_kats(tmp_path):
    """Every reference failure mode is a FormatError (the reference's quik::FormatError)."""
    m = q()
    with pytest.raises(m.FormatError):
        m.load_layer(tmp_path / "missing")  # test_runtime.cpp:481
    cases = {
        "format": lambda j: j["metadata"].__setitem__("format", "something-else"),
        "dtype": lambda j: j["tensors"][1].__setitem__("dtype", "f64"),                     # test_container.cpp:95
        "nbytes": lambda j: j["tensors"][1].__setitem__("nbytes", j["tensors"][1]["nbytes"] + 4),  # :99
        "offset": lambda j: j["tensors"][1].__setitem__("offset", j["tensors"][1]["offset"] + 3),  # :103
        "dup": lambda j: j["tensors"][1].__setitem__("name", j["tensors"][0]["name"]),
        "perm": lambda j: j["metadata"].__setitem__("permutation", list(reversed(j["metadata"]["permutation"]))),
        "bits": lambda j: j["metadata"].__setitem__("act_bits", 8),
        "idx": lambda j: j["metadata"].__setitem__("outlier_indices", [0, 0]),
        "missing_tensor": lambda j: j.__setitem__("tensors", j["tensors"][1:]),
        "no_list": lambda j: j.pop("tensors"),
    }
    for name, fn in cases.items():
        d = _bundle(tmp_path, name)
        _patch(d, fn)
        with pytest.raises(m.FormatError):
            m.load_layer(d)
    # truncated blob (test_container.cpp:70-77)
    d = _bundle(tmp_path, "trunc")
    blob = d / "tensors.bin"
    blob.write_bytes(blob.read_bytes()[:7])
    with pytest.raises(m.FormatError):
        m.load_layer(d)
    # malformed JSON
    d = _bundle(tmp_path, "json")
    (d / "manifest.json").write_text("{\"tensors\": [")
    with pytest.raises(m.FormatError):
        m.load_layer(d)
    # an untouched bundle still loads
    assert m.load_layer(_bundle(tmp_path, "ok")).in_features() == 40
