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
