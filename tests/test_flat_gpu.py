"""GPU FlatIndex (index_flat.cpp:22-43) vs the oracle: bit-exact ids, f32
scores and scanned; masked ids never returned; the reference's errors."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ra():
    import paper_2409_10516_b200 as ra
    return ra


@pytest.mark.parametrize("n,d,k,masked", [(500, 16, 10, 0), (3000, 32, 100, 300),
                                          (2048, 128, 100, 640), (64, 8, 64, 0),
                                          (70000, 64, 100, 640)])
def test_flat_matches_oracle(port, n, d, k, masked):
    ra = _ra()
    rng = np.random.default_rng(n + d)
    keys = rng.standard_normal((n, d)).astype(np.float32)
    Q = rng.standard_normal((5, d)).astype(np.float32)
    mask = np.sort(rng.choice(n, size=masked, replace=False)).astype(np.uint32) if masked else None
    flat = ra.FlatIndex(ra.KVGroup(keys))
    res = flat.search_batch(Q, k, mask)
    for qi in range(len(Q)):
        ref = port.flat_search(keys, Q[qi], k, mask)
        np.testing.assert_array_equal(res[qi].ids, ref.ids)
        np.testing.assert_array_equal(res[qi].scores, ref.scores)
        assert res[qi].scanned == ref.scanned == n - masked
        if mask is not None:
            assert not set(res[qi].ids.tolist()) & set(mask.tolist())


def test_flat_ties_break_by_id(port):
    ra = _ra()
    keys = np.tile(np.array([[1, 2, 3, 4]], np.float32), (40, 1))
    keys[7] *= 2
    q = np.ones(4, np.float32)
    r = ra.FlatIndex(ra.KVGroup(keys)).search(q, 5)
    ref = port.flat_search(keys, q, 5)
    assert list(r.ids) == list(ref.ids) == [7, 0, 1, 2, 3]


def test_flat_errors():
    # index_flat.cpp:17-20,24-26 (test_index_flat.cpp)
    ra = _ra()
    keys = np.random.default_rng(3).standard_normal((10, 4)).astype(np.float32)
    f = ra.FlatIndex(ra.KVGroup(keys))
    with pytest.raises(ra.InvalidArgument, match="^k out of range after masking$"):
        f.search(np.ones(4, np.float32), 0)
    with pytest.raises(ra.InvalidArgument, match="^k out of range after masking$"):
        f.search(np.ones(4, np.float32), 9, np.arange(2, dtype=np.uint32))
    with pytest.raises(ra.InvalidArgument, match="^query dimension mismatch$"):
        f.search(np.ones(3, np.float32), 1)
