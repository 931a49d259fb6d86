"""fvecs ingest straight into device memory (rnndg_load_fvecs, SURVEY 8(f)
item 3): the device store equals rnnd::load_fvecs + set_data (builds from it
are byte-identical), and malformed files fail with the reference's messages
(dataset.cpp:55-95, mirrored host-side by evaluate.load_fvecs)."""
import numpy as np
import pytest

from vecs_cases import FVECS_CASES, make_fvecs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    from paper_2310_20419_b200 import rnnd
    return rnnd


@pytest.mark.parametrize("n,d", [(1, 1), (257, 3), (3000, 128), (21000, 960)])
def test_device_store_equals_host_store(R, tmp_path, n, d):
    """21000 x 960 spans three 32 MB staging chunks."""
    from paper_2310_20419_b200 import evaluate as E
    data = np.random.default_rng(n + d).random((n, d), dtype=np.float32)
    p = str(tmp_path / "x.fvecs")
    E.write_fvecs(R.VectorStore(data), p)
    dev = R.Device()
    ds = dev.load_fvecs(p)
    assert (ds.n, ds.d) == (n, d)
    if n < 3:
        return
    params = R.BuildParams(S=min(10, n - 1), R=12, T1=2, T2=2)
    g_dev = R.build(ds, params)
    g_host = R.build(R.VectorStore(data), params)
    assert R.index_bytes(g_dev) == R.index_bytes(g_host)
    q = R.VectorStore(data[:7])
    a = R.batch_search(g_dev, ds, q, R.SearchParams(L=16, k=3))
    b = R.batch_search(g_host, R.VectorStore(data), q, R.SearchParams(L=16, k=3))
    assert [r.ids.tolist() for r in a] == [r.ids.tolist() for r in b]


@pytest.mark.parametrize("name,records", FVECS_CASES[1:], ids=[c[0] for c in FVECS_CASES[1:]])
def test_malformed_files_match_reference_messages(R, tmp_path, name, records):
    from paper_2310_20419_b200 import evaluate as E
    p = str(tmp_path / f"{name}.fvecs")
    make_fvecs(p, name, records)
    with pytest.raises(R.DataError) as host:
        E.load_fvecs(p)
    with pytest.raises(R.DataError) as dev:
        R.Device().load_fvecs(p)
    assert str(dev.value) == str(host.value)


def test_missing_file(R, tmp_path):
    with pytest.raises(R.DataError, match="cannot open"):
        R.Device().load_fvecs(str(tmp_path / "nope.fvecs"))


@pytest.mark.parametrize("name,records", FVECS_CASES[1:], ids=[c[0] for c in FVECS_CASES[1:]])
def test_failed_load_leaves_no_store(R, tmp_path, name, records):
    """A malformed file after a good one: the context keeps neither the old
    store nor its graph (no half-overwritten rows, no freed buffer): the next
    build fails with ParamError instead of reading stale memory."""
    from paper_2310_20419_b200 import evaluate as E
    good = str(tmp_path / "good.fvecs")
    E.write_fvecs(R.VectorStore(np.random.default_rng(0).random((300, 8), dtype=np.float32)),
                  good)
    bad = str(tmp_path / f"{name}.fvecs")
    make_fvecs(bad, name, records)
    dev = R.Device()
    ds = dev.load_fvecs(good)
    R.build(ds, R.BuildParams(S=10, R=12, T1=1, T2=2))
    with pytest.raises(R.DataError):
        dev.load_fvecs(bad)
    with pytest.raises(R.ParamError, match="no vector data"):
        R.build(ds, R.BuildParams(S=10, R=12, T1=1, T2=2))


def test_whole_graph_calls_rejected_on_a_shard(R):
    """After rnndg_set_partition the whole-graph entry points return
    RNNDG_EPARAM instead of indexing [0, n) arrays of an nv-sized shard."""
    import ctypes as C
    from paper_2310_20419_b200 import _lib
    data = np.random.default_rng(1).random((400, 8), dtype=np.float32)
    dev = R.Device()
    dev.set_data(R.VectorStore(data))
    L, h = dev._L, dev.h
    assert L.rnndg_set_partition(h, 100, 300) == _lib.OK
    assert L.rnndg_random_init(h, 8, 3) == _lib.OK
    c = _lib.Counts()
    assert L.rnndg_update_pass(h, C.byref(c)) == _lib.EPARAM
    assert L.rnndg_reverse(h, 8, 0) == _lib.EPARAM
    assert L.rnndg_sort_lists(h) == _lib.EPARAM
    out = np.zeros(3, np.uint64)
    assert L.rnndg_degree_stats(h, 0, _lib.ptr(out, _lib.u64p)) == _lib.EPARAM
    size = C.c_uint64()
    assert L.rnndg_index_bytes(h, None, C.byref(size)) == _lib.EPARAM
    assert L.rnndg_build(h, 8, 8, 1, 1, 42, 0, None, _lib.PROGRESS_FN(), None) == _lib.EPARAM
    assert b"partitioned" in L.rnndg_last_error(h)
    # the shard protocol itself still runs
    n = C.c_uint64()
    assert L.rnndg_shard_scan(h, C.byref(c), C.byref(n)) == _lib.OK
