"""The tier oracle (oracle/_ref RefCache = the reference TieredKvCache behind
ref_shim.cpp) pinned to the reference's own kv_store test cases
(test_kv_store.cpp:47-110, block size 4, dim 2) before it judges K5."""
import numpy as np
import pytest

import py_oracle as P

pytestmark = pytest.mark.skipif(P.ref() is None, reason="oracle/_ref not built")


def _block(c, layer, base):
    for i in range(4):
        c.append_token(layer, np.array([base + i, -base]), np.array([base, base]))


def test_eviction_lru_lower_id_on_ties():
    c = P.RefCache(1, 2, 2, block_size=4)
    _block(c, 0, 10.0), _block(c, 0, 20.0), _block(c, 0, 30.0)
    assert c.state(0)[0].tolist() == [0, 1, 1]
    c.mark_selected(0, [1], 5)
    _block(c, 0, 40.0)
    assert c.state(0)[0].tolist() == [0, 1, 0, 1]


def test_recall_visibility_and_rejections():
    c = P.RefCache(2, 2, 2, block_size=4)
    for b in (10.0, 20.0, 30.0):
        _block(c, 0, b)
    c.begin_layer(1, 0)
    c.schedule_recall(0, [0], 1, 0)
    assert 0 not in c.residency_set(0).tolist()
    assert c.begin_layer(1, 1) == 0
    assert 0 in c.residency_set(0).tolist() and c.state(0)[0][0] == 0
    c.mark_selected(0, [0, 2], 1)
    assert c.begin_layer(2, 0) == 1
    assert c.state(0)[0].tolist() == [1, 0, 1]
    with pytest.raises(ValueError):
        c.schedule_recall(0, [], 2, 0)
    with pytest.raises(ValueError):
        c.schedule_recall(0, [0], 2, 0)  # already fast
