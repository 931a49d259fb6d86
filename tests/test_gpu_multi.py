"""rnndg_sharded_* (csrc/multi.cu): the vertex-sharded build driven by the
library itself over several device contexts in one process -- identical graph
and per-pass counts to the single-context rnndg_build, for 1..4 shards
(sharing the one GPU of the test box), both prune orders, a d % 4 tail and a
d = 960 C3 prefix; with the fused exchange (records stored straight into the
owner's buffers by rnndg_shard_push, the default) and with the older sorted
export + peer copies (RNNDG_MULTI_EXCHANGE=copy)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _single(R, data, T1, T2, order):
    dev = R.Device()
    dev.set_data(R.VectorStore(data))
    st = R.BuildStats()
    g = R.build(R.VectorStore(data),
                R.BuildParams(S=20, R=40, T1=T1, T2=T2, prune_order=R.PruneOrder(order)),
                st, device=dev)
    counts = [[c.removed, c.inserted, c.flag_skips, c.pair_checks] for c in st.pass_counts]
    return dev.get_graph(), counts


@pytest.fixture(params=["push", "copy"])
def exchange(request):
    old = os.environ.get("RNNDG_MULTI_EXCHANGE")
    os.environ["RNNDG_MULTI_EXCHANGE"] = request.param  # read at every exchange
    yield request.param
    if old is None:
        del os.environ["RNNDG_MULTI_EXCHANGE"]
    else:
        os.environ["RNNDG_MULTI_EXCHANGE"] = old


@pytest.mark.parametrize("shards", [1, 2, 3, 4])
@pytest.mark.parametrize("case", ["uniform67", "c3prefix"])
def test_sharded_build_equals_single(shards, case, exchange):
    import datagen
    from oracle import oracle as O
    from paper_2310_20419_b200 import rnnd as R
    from paper_2310_20419_b200.sharded import MultiDevice
    data = O.synth_uniform(3000, 67, 11) if case == "uniform67" else datagen.rows(3, 3, 0, 2000)
    order = 0 if shards % 2 else 1
    g1, c1 = _single(R, data, 3, 4, order)
    md = MultiDevice([0] * shards)
    md.set_data(data)
    st, c2 = md.build(S=20, R=40, T1=3, T2=4, order=order)
    assert c2 == c1, "per-pass counts differ from rnndg_build"
    assert st.update_passes == 12 and st.reverse_phases == 2
    g2 = md.get_graph()
    assert np.array_equal(g2.offsets, g1.offsets)
    assert np.array_equal(g2.ids, g1.ids)
    assert np.array_equal(g2.dists.view(np.uint32), g1.dists.view(np.uint32))
    assert np.array_equal(g2.fresh, g1.fresh)
    md.close()


def test_sharded_validates():
    from paper_2310_20419_b200 import rnnd as R
    from paper_2310_20419_b200.sharded import MultiDevice
    md = MultiDevice([0, 0])
    with pytest.raises(R.ParamError):
        md.build()
    md.set_data(np.random.default_rng(0).random((50, 8), dtype=np.float32))
    with pytest.raises(R.ParamError):
        md.build(S=60)
    with pytest.raises(Exception):
        MultiDevice([999])


def test_sharded_push_many_shards_larger():
    """7 shards over a 60k-row C5 prefix (d = 96): uneven ownership ranges,
    many records per exchange, every shard pushing into every other's
    buffers concurrently (one host thread per shard)."""
    import datagen
    from paper_2310_20419_b200 import rnnd as R
    from paper_2310_20419_b200.sharded import MultiDevice
    data = datagen.rows(5, 1, 0, 60000)
    g1, c1 = _single(R, data, 2, 3, 0)
    md = MultiDevice([0] * 7)
    md.set_data(data)
    st, c2 = md.build(S=20, R=40, T1=2, T2=3, order=0)
    assert c2 == c1
    g2 = md.get_graph()
    assert np.array_equal(g2.offsets, g1.offsets)
    assert np.array_equal(g2.ids, g1.ids)
    assert np.array_equal(g2.dists.view(np.uint32), g1.dists.view(np.uint32))
    md.close()
