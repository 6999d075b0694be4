"""CPU tests of the host-side mirror of the reference API (paper_2310_09259_b200.quik):
packing, outlier sets and layer validation follow the reference semantics
(packed.cpp, calibration.cpp, runtime.cpp), checked against the oracle."""
import numpy as np
import pytest

import paper_2310_09259_b200 as q
from oracle_lib import oracle


def test_pack_values_matches_oracle_and_reference_layout():
    o = oracle()
    rng = np.random.default_rng(3)
    for bits in (4, 8):
        lim = 7 if bits == 4 else 127
        for (r, c) in [(1, 1), (3, 7), (5, 64), (2, 33)]:
            v = rng.integers(-lim - 1, lim + 1, size=(r, c))
            m = q.pack_values(v, r, c, bits)
            _, ref_bytes = o.pack(v, r, c, bits)
            assert np.array_equal(m.data, ref_bytes)
            assert np.array_equal(q.unpack_values(m), v.astype(np.int8))
            assert m.get(r - 1, c - 1) == v[r - 1, c - 1]
    m = q.pack_values([-8, 7, 0, -1], 1, 4, 4)
    assert list(m.data) == [0xF0, 0x78]


def test_pack_values_range_error_names_row():
    with pytest.raises(IndexError, match="row 1"):
        q.pack_values([0, 0, 8, 0], 2, 2, 4)
    with pytest.raises(ValueError):
        q.pack_values([0, 0], 1, 2, 5)


def test_outlier_set_from_indices():
    o = q.OutlierSet.from_indices(4, [3, 1])
    assert list(o.indices) == [1, 3] and list(o.permutation) == [0, 2, 1, 3]
    assert o.base_count() == 2 and o.outlier_count() == 2
    with pytest.raises(ValueError):
        q.OutlierSet.from_indices(4, [4])
    with pytest.raises(ValueError):
        q.OutlierSet.from_indices(4, [1, 1])
    _, perm = oracle().permutation(10, np.array([0, 5, 9]))
    assert list(q.OutlierSet.from_indices(10, [9, 0, 5]).permutation) == list(perm)


def test_layer_validate_mirrors_reference():
    w = q.QuantizedWeights(q.pack_values(np.zeros((2, 3)), 2, 3, 4), np.ones(2, np.float32),
                           np.zeros((2, 1), np.float32), np.zeros(2, np.float32))
    L = q.QuikLinearLayer(w, q.OutlierSet.from_indices(4, [2]), None, 4)
    L.validate()
    with pytest.raises(ValueError):  # runtime.cpp:151-154
        q.QuikLinearLayer(w, q.OutlierSet.from_indices(4, [1, 2]), None, 4).validate()
    with pytest.raises(ValueError):  # bias length
        q.QuikLinearLayer(w, q.OutlierSet.from_indices(4, [2]), np.zeros(3), 4).validate()
    with pytest.raises(ValueError):  # act bits must match weight bits in quik mode
        q.QuikLinearLayer(w, q.OutlierSet.from_indices(4, [2]), None, 8).validate()
