"""The device segmented sort (build.cu k_seg_sort_warp / k_seg_sort_block),
through rnndg_set_graph, which sorts every imported list nearest-first
(graph.cpp:25-27 order: distance, then id).  Segment lengths straddle every
path: registers (<= 32), warp shared memory (<= 256), CTA shared memory
(<= 4096) and the in-place global-memory network beyond, with distance ties
and non-power-of-two lengths."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LENS = [1, 2, 3, 31, 32, 33, 63, 64, 65, 200, 255, 256, 257, 1000, 4095, 4096, 4097, 9000]


def test_set_graph_sorts_every_segment_length():
    from paper_2310_20419_b200 import rnnd as R
    n = 12000
    rng = np.random.default_rng(3)
    data = rng.random((n, 8), dtype=np.float32)
    lens = np.zeros(n, np.int64)
    lens[:len(LENS)] = LENS
    lens[len(LENS):] = rng.integers(0, 40, n - len(LENS))
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(lens)
    ids, dists = [], []
    for u in range(n):
        m = int(lens[u])
        cand = rng.choice(np.delete(np.arange(n), u), m, replace=False).astype(np.uint32)
        # coarse distances: many ties, broken by id
        dists.append((rng.integers(0, 16, m) / 4.0).astype(np.float32))
        ids.append(cand)
    ids = np.concatenate(ids)
    dists = np.concatenate(dists)
    fresh = rng.integers(0, 2, len(ids)).astype(np.uint8)
    dev = R.Device()
    dev.set_data(R.VectorStore(data))
    dev.set_graph(R.CSR(off, ids, dists, fresh), True)
    g = dev.get_graph()
    assert np.array_equal(g.offsets.astype(np.int64), off.astype(np.int64))
    for u in range(n):
        a, b = int(off[u]), int(off[u + 1])
        order = np.lexsort((ids[a:b], dists[a:b]))
        assert np.array_equal(g.ids[a:b], ids[a:b][order]), u
        assert np.array_equal(g.dists[a:b], dists[a:b][order]), u
        assert np.array_equal(g.fresh[a:b], fresh[a:b][order]), u
