"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
reference-generated golden fixtures.  Bit-exact throughout: distances,
per-pass EditCounts, graph state (ids, dists, fresh flags) and index bytes.
"""
import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

from golden_data import data_for

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def R():
    from paper_2310_20419_b200 import rnnd
    return rnnd


def dev_graph(R, data):
    d = R.Device()
    store = R.VectorStore(data)
    d.set_data(store)
    return d, store


def dev_csr(d):
    from oracle.oracle import CSR
    c = d.get_graph()
    return CSR(c.offsets, c.ids, c.dists, c.fresh)


def counts_of(c):
    return [int(c.removed), int(c.inserted), int(c.flag_skips), int(c.pair_checks)]


# ------------------------------------------------------------------- K1

@pytest.mark.parametrize("d", list(range(1, 68)) + [96, 128, 960])
def test_l2_bit_exact(R, oracle, d):
    rng = np.random.default_rng(1000 + d)
    n = 64
    data = ((rng.random((n, d)) - 0.5) * 8).astype(np.float32)
    data[3] *= np.float32(1e-20)  # subnormal differences must survive (no FTZ)
    data[4] = data[5]  # exact zero distance
    dev, store = dev_graph(R, data)
    a = rng.integers(0, n, 500).astype(np.uint32)
    b = rng.integers(0, n, 500).astype(np.uint32)
    out = np.zeros(500, np.float32)
    from paper_2310_20419_b200._lib import f32p, ptr, u32p
    dev.check(dev._L.rnndg_l2_pairs(dev.h, ptr(a, u32p), ptr(b, u32p), 500, ptr(out, f32p)))
    want = np.array([oracle.l2_sq(data[i], data[j]) for i, j in zip(a, b)], np.float32)
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32))


# ------------------------------------------------------------------- K2

@pytest.mark.parametrize("n,d,S,seed", [(50, 5, 7, 11), (2, 3, 1, 9), (300, 6, 10, 5),
                                        (1000, 128, 20, 42), (129, 960, 64, 1),
                                        (200, 4, 100, 3), (70, 2, 69, 8)])
def test_random_init_identical(R, oracle, n, d, S, seed):
    data = oracle.synth_uniform(n, d, seed + 1)
    dev, _ = dev_graph(R, data)
    dev.check(dev._L.rnndg_random_init(dev.h, S, seed))
    og = oracle.OracleGraph(data)
    assert og.random_init(S, seed) == 0
    # the device keeps every list sorted by (dist, id) (set semantics)
    a, b = dev_csr(dev), og.export().canonical()
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.ids, b.ids)
    assert np.array_equal(a.dists.view(np.uint32), b.dists.view(np.uint32))
    assert np.all(a.fresh == 1)


def test_random_init_param_errors(R, oracle):
    dev, _ = dev_graph(R, oracle.synth_uniform(10, 2, 1))
    with pytest.raises(R.ParamError):
        dev.check(dev._L.rnndg_random_init(dev.h, 0, 1))
    with pytest.raises(R.ParamError):
        dev.check(dev._L.rnndg_random_init(dev.h, 10, 1))
    dev1, _ = dev_graph(R, oracle.synth_uniform(1, 2, 1))
    with pytest.raises(R.ParamError):
        dev1.check(dev1._L.rnndg_random_init(dev1.h, 1, 1))


# ------------------------------------------------------- K3/K4/K5 passes

STEP_CASES = [
    ("uniform", 300, 6, 13, 10, 16, 0),
    ("uniform", 1000, 5, 21, 8, 12, 1),
    ("grid", 800, 2, 4, 12, 10, 0),
    ("grid", 600, 3, 5, 6, 5, 1),
    ("cfg3", 1200, 960, 3, 20, 96, 0),
    ("cfg2", 2000, 128, 2, 20, 96, 0),
]


def step_data(oracle, kind, n, d, s):
    if kind == "uniform":
        return oracle.synth_uniform(n, d, s)
    if kind == "grid":
        return (np.round(oracle.synth_uniform(n, d, s) * 8.0) / 8.0).astype(np.float32)
    import datagen
    return datagen.rows(int(kind[-1]), s, 0, n)


@pytest.mark.parametrize("case", STEP_CASES, ids=[f"{c[0]}-{c[1]}x{c[2]}" for c in STEP_CASES])
def test_pass_by_pass_parity(R, oracle, case):
    """Every update pass and reverse phase leaves identical state and counts."""
    kind, n, d, s, S, Rcap, order = case
    data = step_data(oracle, kind, n, d, s)
    dev, _ = dev_graph(R, data)
    dev.check(dev._L.rnndg_random_init(dev.h, S, 7))
    og = oracle.OracleGraph(data)
    og.random_init(S, 7)
    from paper_2310_20419_b200 import _lib
    for t1 in range(3):
        for t2 in range(4):
            c = _lib.Counts()
            dev.check(dev._L.rnndg_update_pass(dev.h, C.byref(c)))
            want = og.update_pass().tolist()
            assert counts_of(c) == want, (t1, t2)
            assert dev_csr(dev).same_as(og.export()), (t1, t2)
        dev.check(dev._L.rnndg_reverse(dev.h, Rcap, order))
        assert og.add_reverse_edges(Rcap, order) == 0
        assert dev_csr(dev).same_as(og.export()), ("reverse", t1)


def test_big_lists_parity(R, oracle):
    """Lists far longer than a warp (a hub with 3,000 entries and long tails)
    go through the same sort / scan / apply path."""
    n, d = 4000, 8
    data = oracle.synth_uniform(n, d, 77)
    rng = np.random.default_rng(5)
    lists = []
    for u in range(n):
        m = 3000 if u == 0 else (400 if u % 97 == 0 else 12)
        ids = rng.choice(np.delete(np.arange(n), u), m, replace=False).astype(np.uint32)
        lists.append(ids)
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(l) for l in lists])
    ids = np.concatenate(lists).astype(np.uint32)
    owner = np.repeat(np.arange(n), [len(l) for l in lists])
    dists = np.array([oracle.l2_sq(data[u], data[v]) for u, v in zip(owner, ids)], np.float32)
    fresh = (rng.random(len(ids)) < 0.5).astype(np.uint8)
    from oracle.oracle import CSR
    csr = CSR(off, ids, dists, fresh)
    dev, _ = dev_graph(R, data)
    dev.set_graph(R.CSR(off, ids, dists, fresh), True)
    og = oracle.OracleGraph(data)
    og.load(csr)
    from paper_2310_20419_b200 import _lib
    for _ in range(3):
        c = _lib.Counts()
        dev.check(dev._L.rnndg_update_pass(dev.h, C.byref(c)))
        assert counts_of(c) == og.update_pass().tolist()
        assert dev_csr(dev).same_as(og.export())
    dev.check(dev._L.rnndg_reverse(dev.h, 50, 0))
    og.add_reverse_edges(50, 0)
    assert dev_csr(dev).same_as(og.export())


# ------------------------------------------------------------ full build

def load_cases():
    with open(os.path.join(GOLDEN, "builds.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", load_cases(),
                         ids=lambda c: f"{c['kind']}{c.get('cfg', '')}-{c['n']}x{c['d']}")
def test_build_matches_reference_fixture(R, case):
    """rnnd::build(threads=4) golden: index bytes and every per-pass count."""
    data = data_for(case)
    assert hashlib.sha256(data.tobytes()).hexdigest() == case["data_sha256"]
    store = R.VectorStore(data)
    st = R.BuildStats()
    p = R.BuildParams(S=case["S"], R=case["R"], T1=case["T1"], T2=case["T2"],
                      seed=case["seed"], prune_order=R.PruneOrder(case["order"]))
    g = R.build(store, p, st)
    assert [[c.removed, c.inserted, c.flag_skips, c.pair_checks] for c in st.pass_counts] \
        == case["per_pass"]
    assert [st.edits.removed, st.edits.inserted, st.edits.flag_skips,
            st.edits.pair_checks] == case["edits"]
    assert hashlib.sha256(R.index_bytes(g)).hexdigest() == case["index_sha256"]
    assert st.update_passes == case["T1"] * case["T2"]
    assert st.reverse_phases == case["T1"] - 1
    assert st.seconds > 0


@pytest.mark.slow
def test_build_c1_prefix_vs_oracle(R, oracle):
    import datagen
    data = datagen.rows(1, 0, 0, 8000)
    g = R.build(R.VectorStore(data))
    og = oracle.OracleGraph(data)
    og.build()
    assert R.index_bytes(g) == og.index_bytes()


def test_build_structure_and_progress(R, oracle):  # test_builder.cpp:255-284
    store = R.VectorStore(oracle.synth_uniform(150, 4, 3))
    calls = []
    st = R.BuildStats()
    g = R.build(store, R.BuildParams(S=6, R=10, T1=3, T2=2), st,
                lambda t1, T1, outer, el: calls.append((t1, T1, el)))
    assert st.update_passes == 6 and st.reverse_phases == 2 and len(calls) == 3
    assert all(t1 <= T1 for t1, T1, _ in calls)
    for u in range(g.size()):
        l = g.list(u)
        assert all((a.dist, a.id) < (b.dist, b.id) for a, b in zip(l, l[1:]))
        assert len({e.id for e in l}) == len(l) and all(e.id != u for e in l)
    R.build(store, R.BuildParams(S=6, R=10, T1=1, T2=4), st)
    assert st.reverse_phases == 0 and st.update_passes == 4


def test_build_validates(R, oracle):  # test_builder.cpp:286-297
    store = R.VectorStore(oracle.synth_uniform(10, 3, 1))
    for kw in (dict(S=10), dict(S=2, T1=0), dict(S=2, R=0), dict(S=0)):
        with pytest.raises(R.ParamError):
            R.build(store, R.BuildParams(**kw))


# -------------------------------------------------- hand cases (mirror API)

def line(xs):
    return np.array(xs, np.float32).reshape(-1, 1)


def E(R, oracle, s, a, b, fresh):
    return R.NeighborEntry(b, oracle.l2_sq(s[a], s[b]), fresh)


def test_update_redirect_hand_case(R, oracle):  # test_builder.cpp:104-123
    s = line([0.0, 1.0, 1.5])
    store = R.VectorStore(s)
    g = R.AdjacencyGraph.from_lists([[E(R, oracle, s, 0, 1, True), E(R, oracle, s, 0, 2, True)],
                                     [], []])
    ec = R.update_neighbors(g, store, 1)
    assert (ec.removed, ec.inserted, ec.pair_checks, ec.flag_skips) == (1, 1, 1, 0)
    assert [(e.id, e.fresh) for e in g.list(0)] == [(1, False)]
    assert [e.id for e in g.list(1)] == [2] and g.list(1)[0].dist == oracle.l2_sq(s[1], s[2])
    assert g.list(2) == []


def test_old_old_skip_hand_case(R, oracle):  # test_builder.cpp:125-143
    s = line([0.0, 1.0, 1.75])
    store = R.VectorStore(s)
    g = R.AdjacencyGraph.from_lists([[E(R, oracle, s, 0, 1, False), E(R, oracle, s, 0, 2, False)],
                                     [], []])
    ec = R.update_neighbors(g, store)
    assert (ec.removed, ec.inserted, ec.pair_checks, ec.flag_skips) == (0, 0, 0, 1)
    assert len(g.list(0)) == 2
    g.set_lists([[E(R, oracle, s, 0, 1, False), E(R, oracle, s, 0, 2, True)], [], []])
    ec = R.update_neighbors(g, store)
    assert ec.removed == 1 and ec.pair_checks == 1 and len(g.list(0)) == 1


def test_no_duplicate_redirect(R, oracle):  # test_builder.cpp:145-156
    s = line([0.0, 1.0, 1.75])
    store = R.VectorStore(s)
    g = R.AdjacencyGraph.from_lists([[E(R, oracle, s, 0, 1, True), E(R, oracle, s, 0, 2, True)],
                                     [E(R, oracle, s, 1, 2, False)], []])
    ec = R.update_neighbors(g, store)
    assert ec.removed == 1 and ec.inserted == 0 and [e.id for e in g.list(1)] == [2]


def test_update_requires_distances(R):  # test_builder.cpp:158-163
    g = R.AdjacencyGraph.from_lists([[], []], has_distances=False)
    with pytest.raises(R.ParamError):
        R.update_neighbors(g, R.VectorStore(line([0.0, 1.0])))


@pytest.mark.parametrize("order", [R_ for R_ in (0, 1)])
def test_reverse_star_hand_case(R, oracle, order):  # test_builder.cpp:187-209
    s = line([0.0, 1.0, 2.0, 3.0, 4.0, 5.0])
    g = R.AdjacencyGraph.from_lists([[]] + [[E(R, oracle, s, i, 0, False)] for i in range(1, 6)])
    R.add_reverse_edges(g, 3, 1, R.PruneOrder(order), store=R.VectorStore(s))
    assert sorted(e.id for e in g.list(0)) == [1, 2, 3] and all(e.fresh for e in g.list(0))
    for i in (1, 2, 3):
        assert [(e.id, e.fresh) for e in g.list(i)] == [(0, False)]
    assert g.list(4) == [] and g.list(5) == []


def test_reverse_validates(R):
    g = R.AdjacencyGraph.from_lists([[], []])
    with pytest.raises(R.ParamError):
        R.add_reverse_edges(g, 0, store=R.VectorStore(line([0.0, 1.0])))


def test_rng_strategy_goldens(R, oracle):  # test_builder.cpp:53-79
    s = line([0.0, 1.0, 1.8, 3.0])
    st = R.VectorStore(s)
    kept = R.rng_strategy(st, 0, [E(R, oracle, s, 0, 2, True), E(R, oracle, s, 0, 1, True),
                                  E(R, oracle, s, 0, 3, True)])
    assert [e.id for e in kept] == [1]
    s2 = line([0.0, 1.0, -1.0])
    kept = R.rng_strategy(R.VectorStore(s2), 0, [E(R, oracle, s2, 0, 1, True),
                                                 E(R, oracle, s2, 0, 2, True)])
    assert [e.id for e in kept] == [1, 2]
    s3 = line([0.0, 1.0])
    assert R.rng_strategy(R.VectorStore(s3), 0, []) == []
    with pytest.raises(R.ParamError):
        R.rng_strategy(R.VectorStore(s3), 0, [E(R, oracle, s3, 0, 1, True),
                                              R.NeighborEntry(0, 0.0, True)])


def test_rng_strategy_random_vs_oracle(R, oracle):  # test_builder.cpp:81-102
    data = oracle.synth_uniform(150, 4, 31)
    st = R.VectorStore(data)
    dev = R.Device()
    rng = np.random.default_rng(7)
    for _ in range(20):
        u = int(rng.integers(150))
        ids = rng.choice(np.delete(np.arange(150), u), 30, replace=False)
        ds = [oracle.l2_sq(data[u], data[i]) for i in ids]
        kept = R.rng_strategy(st, u, [R.NeighborEntry(int(i), d, True) for i, d in zip(ids, ds)],
                              device=dev)
        ki, kd = oracle.rng_strategy(data, u, ids, ds)
        assert [e.id for e in kept] == ki.tolist()


def test_fixed_point_of_built_graph(R, oracle):  # test_builder.cpp:312-323
    data = oracle.synth_uniform(200, 4, 41)
    store = R.VectorStore(data)
    g = R.build(store)
    dev = R.Device()
    for u in range(g.size()):
        lst = g.list(u)
        kept = R.rng_strategy(store, u, lst, device=dev)
        assert [e.id for e in kept] == [e.id for e in lst]


def test_set_graph_validation(R, oracle):  # graph.cpp:152-167 load checks
    store = R.VectorStore(oracle.synth_uniform(4, 2, 1))
    for lists in ([[R.NeighborEntry(1, 1.0, False), R.NeighborEntry(1, 1.0, False)], [], [], []],
                  [[R.NeighborEntry(0, 0.0, False)], [], [], []],
                  [[R.NeighborEntry(9, 1.0, False)], [], [], []]):
        g = R.AdjacencyGraph.from_lists(lists)
        with pytest.raises(R.DataError):
            R.update_neighbors(g, store)


# ---------------------------------------------------------------- search

def test_search_matches_reference_golden(R, oracle):
    """rnnd::batch_search goldens: ids, dists, visited and dist_comps."""
    fx = np.load(os.path.join(GOLDEN, "search.npz"))
    cases = [c for c in load_cases() if c.get("cfg") == 1]
    data = data_for(cases[0])
    import datagen
    q = datagen.rows(1, 0, 3000, 200)
    assert hashlib.sha256(q.tobytes()).digest() == fx["queries_sha256"].tobytes()
    store = R.VectorStore(data)
    g = R.build(store)
    for L, K in [(10, 0), (32, 0), (64, 16), (16, 4)]:
        res = R.batch_search(g, store, R.VectorStore(q), R.SearchParams(L=L, K=K, k=10))
        ids = np.stack([r.ids for r in res])
        dists = np.stack([r.dists for r in res])
        assert np.array_equal(ids, fx[f"ids_L{L}_K{K}"])
        assert np.array_equal(dists.view(np.uint32), fx[f"dists_L{L}_K{K}"].view(np.uint32))
        assert [r.visited for r in res] == fx[f"visited_L{L}_K{K}"].tolist()
        assert [r.dist_comps for r in res] == fx[f"comps_L{L}_K{K}"].tolist()
    gt = R.brute_force_gt(store, R.VectorStore(q), 10)
    assert np.array_equal(gt.ids, fx["gt10"])


@pytest.mark.parametrize("L,K,k,mode", [(8, 0, 3, 0), (40, 5, 5, 0), (100, 0, 10, 0),
                                        (200, 3, 7, 1), (17, 2, 17, 1)])
def test_search_vs_oracle(R, oracle, L, K, k, mode):
    data = oracle.synth_uniform(500, 7, 19)
    store = R.VectorStore(data)
    g = R.build(store, R.BuildParams(S=8, R=16, T1=2, T2=3))
    og = oracle.OracleGraph(data)
    c = g.csr
    from oracle.oracle import CSR
    og.load(CSR(c.offsets, c.ids, c.dists, c.fresh))
    qs = oracle.synth_uniform(30, 7, 20)
    res = R.batch_search(g, store, R.VectorStore(qs),
                         R.SearchParams(L=L, K=K, k=k, entry=R.EntryMode(mode), entry_vertex=3))
    for qi in range(30):
        ids, dists, vis, comps = og.search(qs[qi], L=L, K=K, k=k, entry_mode=mode,
                                           entry_vertex=3)
        assert res[qi].ids.tolist() == ids.tolist()
        assert np.array_equal(res[qi].dists.view(np.uint32), dists.view(np.uint32))
        assert (res[qi].visited, res[qi].dist_comps) == (vis, comps)


def test_search_exhaustive_pool(R, oracle):  # test_search.cpp:28-43
    store = R.VectorStore(oracle.synth_uniform(120, 5, 3))
    qs = R.VectorStore(oracle.synth_uniform(25, 5, 4))
    gt = R.brute_force_gt(store, qs, 3)
    g = R.AdjacencyGraph(120)
    res = R.batch_search(g, store, qs, R.SearchParams(L=120, k=3))
    for q in range(25):
        assert res[q].ids.tolist() == gt.ids[q].tolist()


def test_search_hand_cases(R, oracle):  # test_search.cpp:45-108
    st = np.array([[0, 0], [1, 0], [5, 5]], np.float32)
    g = R.AdjacencyGraph.from_lists([[E(R, oracle, st, 0, 1, False)],
                                     [E(R, oracle, st, 1, 0, False), E(R, oracle, st, 1, 2, False)],
                                     [E(R, oracle, st, 2, 1, False)]])
    r = R.search(g, R.VectorStore(st), np.array([0.9, 0.0], np.float32),
                 R.SearchParams(L=3, k=1))
    assert r.ids.tolist() == [1] and r.visited <= 3 and r.dist_comps <= 3
    s = line([0, 1, 2, 3, 4, 5])
    g = R.AdjacencyGraph.from_lists([[E(R, oracle, s, 0, i, False) for i in range(1, 6)]] +
                                    [[]] * 5)
    p = R.SearchParams(L=6, k=6, K=2, entry=R.EntryMode.kFixedVertex, entry_vertex=0)
    r = R.search(g, R.VectorStore(s), np.zeros(1, np.float32), p)
    assert r.ids.tolist() == [0, 1, 2] and r.visited == 3 and r.dist_comps == 3
    p.K = 0
    assert len(R.search(g, R.VectorStore(s), np.zeros(1, np.float32), p).ids) == 6
    s = line([0.0, 1.0, 100.0, 101.0])
    g = R.AdjacencyGraph.from_lists([[E(R, oracle, s, 0, 1, False)], [E(R, oracle, s, 1, 0, False)],
                                     [E(R, oracle, s, 2, 3, False)], [E(R, oracle, s, 3, 2, False)]])
    r = R.search(g, R.VectorStore(s), np.array([100.5], np.float32),
                 R.SearchParams(L=2, k=1, entry=R.EntryMode.kFixedVertex))
    assert r.ids.tolist() == [1]


def test_search_validates(R, oracle):  # test_search.cpp:110-128
    store = R.VectorStore(oracle.synth_uniform(10, 3, 1))
    g = R.random_init(store, 2, 1)
    q = np.zeros(3, np.float32)
    for p in (R.SearchParams(L=4, k=5), R.SearchParams(L=0, k=1),
              R.SearchParams(L=4, entry=R.EntryMode.kFixedVertex, entry_vertex=10)):
        with pytest.raises(R.ParamError):
            R.search(g, store, q, p)
    with pytest.raises(R.ParamError):
        R.search(g, store, np.zeros(4, np.float32), R.SearchParams(L=4))


def test_brute_force_ties_and_full_sort(R, oracle):  # test_dataset.cpp:156-197
    base = R.VectorStore(np.array([[1, 0], [1, 0], [2, 2]], np.float32))
    assert R.brute_force_gt(base, R.VectorStore(np.zeros((1, 2), np.float32)), 2).ids[0].tolist() \
        == [0, 1]
    b = oracle.synth_uniform(1200, 6, 7)
    q = oracle.synth_uniform(15, 6, 8)
    gt = R.brute_force_gt(R.VectorStore(b), R.VectorStore(q), 9)
    assert np.array_equal(gt.ids, oracle.brute_force(b, q, 9))


def test_recall_tie_rule(R):  # test_eval.cpp:30-58
    base = R.VectorStore(np.array([[0, 0], [0, 0], [5, 5]], np.float32))
    qs = R.VectorStore(np.array([[0.1, 0], [4, 4]], np.float32))
    gt = R.GroundTruth(1, np.array([[0], [2]], np.uint32))
    d0 = R.l2_sq_rows(qs.data[:1], base.data[:1])[0]
    d1 = R.l2_sq_rows(qs.data[1:], base.data[2:])[0]
    res = [R.SearchResult(np.array([1], np.uint32), np.array([d0], np.float32)),
           R.SearchResult(np.array([2], np.uint32), np.array([d1], np.float32))]
    assert R.recall_at_1(res, gt, base, qs) == 1.0


def test_degree_stats_hand_case(R):  # test_graph.cpp:115-135
    g = R.AdjacencyGraph.from_lists([[R.NeighborEntry(1, 2.0, False), R.NeighborEntry(2, 1.0, False)],
                                     [R.NeighborEntry(0, 2.0, False)], []])
    st = R.degree_stats(g)
    assert (st.edges, st.avg_out, st.max_out, st.max_in) == (3, 1.0, 2, 1)
    st = R.degree_stats(g, 1)
    assert (st.edges, st.max_out, st.max_in) == (2, 1, 1)


def test_index_roundtrip(R, oracle, tmp_path):  # test_graph.cpp:174-263
    store = R.VectorStore(oracle.synth_uniform(40, 3, 2))
    g = R.build(store, R.BuildParams(S=5, R=8, T1=2, T2=2))
    p = str(tmp_path / "g.idx")
    R.save_index(g, p)
    back = R.load_index(p)
    assert not back.has_distances
    assert back.csr.ids.tolist() == g.csr.ids.tolist()
    assert R.index_bytes(back) == R.index_bytes(g)
    raw = bytearray(open(p, "rb").read())
    raw[-10] ^= 0x40
    open(p, "wb").write(bytes(raw))
    with pytest.raises(R.DataError, match="checksum"):
        R.load_index(p)
