"""Pin the CPU oracle (oracle/rnnd_oracle.c) before trusting it.

Every golden value below is one the reference's own unit tests assert
(paths relative to /root/reference/proj/tests); the test names cite them.
The oracle is test infrastructure only (see oracle/rnnd_oracle.h).
"""
import hashlib
import json
import os

import numpy as np
import pytest

from golden_data import data_for

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def line(xs):
    return np.array(xs, np.float32).reshape(-1, 1)


def edge(O, data, a, b, fresh):
    return (b, O.l2_sq(data[a], data[b]), 1 if fresh else 0)


def graph_from(O, data, lists):
    """lists[u] = [(id, dist, fresh)]"""
    g = O.OracleGraph(data)
    off = np.zeros(len(lists) + 1, np.uint64)
    for u, l in enumerate(lists):
        off[u + 1] = off[u] + len(l)
    flat = [e for l in lists for e in l]
    csr = O.CSR(off, np.array([e[0] for e in flat], np.uint32),
                np.array([e[1] for e in flat], np.float32),
                np.array([e[2] for e in flat], np.uint8))
    g.load(csr)
    return g


def lists_of(g):
    c = g.export()
    return [[(int(c.ids[j]), float(c.dists[j]), int(c.fresh[j]))
             for j in range(int(c.offsets[u]), int(c.offsets[u + 1]))]
            for u in range(c.n)]


# ---------------------------------------------------------- test_metric.cpp

def test_splitmix_published_sequence(oracle):  # test_metric.cpp:32-39
    import ctypes as C
    s = C.c_uint64(0)
    L = oracle.lib()
    assert L.ro_splitmix_next(C.byref(s)) == 0xE220A8397B1DCDAF
    assert L.ro_splitmix_next(C.byref(s)) == 0x6E789E6AA1B965F4
    assert L.ro_splitmix_next(C.byref(s)) == 0x06C45D188009454F
    s = C.c_uint64(42)
    assert L.ro_splitmix_next(C.byref(s)) == 0xBDD732262FEB6E95


def test_splitmix_derived_draws(oracle):  # test_metric.cpp:41-53
    import ctypes as C
    L = oracle.lib()
    s = C.c_uint64(42)
    assert L.ro_splitmix_bounded(C.byref(s), 10) == 7
    s = C.c_uint64(42)
    assert np.float32(L.ro_splitmix_unit_float(C.byref(s))) == \
        np.float32(0xBDD732262FEB6E95 >> 40) / np.float32(16777216.0)
    s = C.c_uint64(1234)
    for _ in range(1000):
        f = L.ro_splitmix_unit_float(C.byref(s))
        assert 0.0 <= f < 1.0
        assert L.ro_splitmix_bounded(C.byref(s), 17) < 17


def test_sample_distinct_excludes_pivot(oracle):  # test_metric.cpp:55-75
    state = 7
    for n in (5, 50, 300):
        for count in (1, 3, n - 1):
            out, state = oracle.sample_distinct(state, n, count, n // 2)
            assert len(out) == count
            assert len(set(out.tolist())) == count
            assert all(v < n and v != n // 2 for v in out)
    allv, _ = oracle.sample_distinct(state, 100, 100)
    assert sorted(allv.tolist()) == list(range(100))


def test_l2_exact_small_cases(oracle):  # test_metric.cpp:77-89
    assert oracle.l2_sq([0, 0], [3, 4]) == 25.0
    assert oracle.l2_sq([0.5, 0.25, 1.0, -2.0, 3.0], [0] * 5) == 14.3125
    assert oracle.l2_sq([3, 4], [3, 4]) == 0.0


def test_l2_tracks_f64_within_1e6(oracle):  # test_metric.cpp:104-119
    rng = np.random.default_rng(123)
    for d in (1, 2, 3, 8, 33, 128, 301):
        for _ in range(10):
            a = ((rng.random(d) - 0.5) * 2).astype(np.float32)
            b = ((rng.random(d) - 0.5) * 2).astype(np.float32)
            ref = float(np.sum((a.astype(np.float64) - b.astype(np.float64)) ** 2))
            got = oracle.l2_sq(a, b)
            assert (got == 0) if ref == 0 else abs(got - ref) / ref <= 1e-6


def test_l2_symmetry(oracle):  # test_metric.cpp:121-131
    rng = np.random.default_rng(5)
    for _ in range(50):
        a = (rng.random(19) - 0.5).astype(np.float32)
        b = (rng.random(19) - 0.5).astype(np.float32)
        assert oracle.l2_sq(a, b) == oracle.l2_sq(b, a) >= 0


def test_synth_uniform_first_value(oracle):  # test_dataset.cpp:109-123
    a = oracle.synth_uniform(20, 7, 42)
    assert a[0, 0] == np.float32(0xBDD732262FEB6E95 >> 40) / np.float32(16777216.0)
    assert np.array_equal(a, oracle.synth_uniform(20, 7, 42))
    assert not np.array_equal(a, oracle.synth_uniform(20, 7, 43))
    assert a.min() >= 0 and a.max() < 1


# --------------------------------------------------------- test_builder.cpp

def test_rng_strategy_drops_occluded(oracle):  # test_builder.cpp:53-61
    s = line([0.0, 1.0, 1.8, 3.0])
    cand = [edge(oracle, s, 0, 2, 1), edge(oracle, s, 0, 1, 1), edge(oracle, s, 0, 3, 1)]
    ki, _ = oracle.rng_strategy(s, 0, [c[0] for c in cand], [c[1] for c in cand])
    assert ki.tolist() == [1]


def test_rng_strategy_mutually_visible(oracle):  # test_builder.cpp:63-72
    s = line([0.0, 1.0, -1.0])
    cand = [edge(oracle, s, 0, 1, 1), edge(oracle, s, 0, 2, 1)]
    ki, _ = oracle.rng_strategy(s, 0, [c[0] for c in cand], [c[1] for c in cand])
    assert ki.tolist() == [1, 2]


def test_rng_strategy_edge_cases(oracle):  # test_builder.cpp:74-79
    s = line([0.0, 1.0])
    ki, _ = oracle.rng_strategy(s, 0, [], [])
    assert len(ki) == 0
    with pytest.raises(ValueError):
        oracle.rng_strategy(s, 0, [1, 0], [1.0, 0.0])


def test_update_pass_redirects(oracle):  # test_builder.cpp:104-123
    s = line([0.0, 1.0, 1.5])
    g = graph_from(oracle, s, [[edge(oracle, s, 0, 1, 1), edge(oracle, s, 0, 2, 1)], [], []])
    c = g.update_pass()
    assert c.tolist() == [1, 1, 0, 1]  # removed, inserted, flag_skips, pair_checks
    L = lists_of(g)
    assert [(e[0], e[2]) for e in L[0]] == [(1, 0)]
    assert [e[0] for e in L[1]] == [2]
    assert L[1][0][1] == oracle.l2_sq(s[1], s[2])
    assert L[2] == []


def test_old_old_skip(oracle):  # test_builder.cpp:125-143
    s = line([0.0, 1.0, 1.75])
    g = graph_from(oracle, s, [[edge(oracle, s, 0, 1, 0), edge(oracle, s, 0, 2, 0)], [], []])
    c = g.update_pass()
    assert c.tolist() == [0, 0, 1, 0]
    assert len(lists_of(g)[0]) == 2
    g = graph_from(oracle, s, [[edge(oracle, s, 0, 1, 0), edge(oracle, s, 0, 2, 1)], [], []])
    c = g.update_pass()
    assert c[0] == 1 and c[3] == 1
    assert len(lists_of(g)[0]) == 1


def test_redirect_not_duplicated(oracle):  # test_builder.cpp:145-156
    s = line([0.0, 1.0, 1.75])
    g = graph_from(oracle, s, [[edge(oracle, s, 0, 1, 1), edge(oracle, s, 0, 2, 1)],
                               [edge(oracle, s, 1, 2, 0)], []])
    c = g.update_pass()
    assert c[0] == 1 and c[1] == 0
    assert [e[0] for e in lists_of(g)[1]] == [2]


@pytest.mark.parametrize("order", [0, 1])
def test_reverse_star(oracle, order):  # test_builder.cpp:187-209
    s = line([0.0, 1.0, 2.0, 3.0, 4.0, 5.0])
    lists = [[]] + [[edge(oracle, s, i, 0, 0)] for i in range(1, 6)]
    g = graph_from(oracle, s, lists)
    assert g.add_reverse_edges(3, order) == 0
    L = lists_of(g)
    assert sorted(e[0] for e in L[0]) == [1, 2, 3]
    assert all(e[2] == 1 for e in L[0])
    for i in (1, 2, 3):
        assert [(e[0], e[2]) for e in L[i]] == [(0, 0)]
    assert L[4] == [] and L[5] == []


def test_reverse_mutual_dedup(oracle):  # test_builder.cpp:211-220
    s = line([0.0, 1.0])
    g = graph_from(oracle, s, [[edge(oracle, s, 0, 1, 0)], [edge(oracle, s, 1, 0, 0)]])
    g.add_reverse_edges(5, 0)
    L = lists_of(g)
    assert g.edges() == 2 and L[0][0][2] == 0 and L[1][0][2] == 0


def test_build_validation(oracle):  # test_builder.cpp:286-297
    data = oracle.synth_uniform(10, 3, 1)
    g = oracle.OracleGraph(data)
    assert g.build(S=10)[0] == 1
    assert g.build(S=2, T1=0)[0] == 1
    assert g.build(S=2, R=0)[0] == 1


def test_fixed_point_of_serial_build(oracle):  # test_builder.cpp:312-323
    data = oracle.synth_uniform(200, 4, 41)
    g = oracle.OracleGraph(data)
    g.build(serial=True)
    c = g.export()
    for u in range(c.n):
        a, b = int(c.offsets[u]), int(c.offsets[u + 1])
        ki, _ = oracle.rng_strategy(data, u, c.ids[a:b], c.dists[a:b])
        assert ki.tolist() == c.ids[a:b].tolist()


# ----------------------------------------------------------- test_graph.cpp

def test_random_init_exact_distances(oracle):  # test_graph.cpp:66-79
    data = oracle.synth_uniform(50, 5, 3)
    g = oracle.OracleGraph(data)
    assert g.random_init(7, 11) == 0
    c = g.export()
    assert np.all(np.diff(c.offsets) == 7)
    for u in range(50):
        ids = c.ids[7 * u:7 * u + 7]
        assert len(set(ids.tolist())) == 7 and u not in ids.tolist()
        for j, v in enumerate(ids):
            assert c.dists[7 * u + j] == oracle.l2_sq(data[u], data[v])
    assert np.all(c.fresh == 1)


def test_random_init_two_points(oracle):  # test_graph.cpp:98-105
    g = oracle.OracleGraph(line([0.0, 1.0]))
    g.random_init(1, 9)
    assert g.export().ids.tolist() == [1, 0]


def test_random_init_validation(oracle):  # test_graph.cpp:107-113
    g = oracle.OracleGraph(oracle.synth_uniform(10, 2, 1))
    assert g.random_init(0, 1) == 1 and g.random_init(10, 1) == 1
    assert oracle.OracleGraph(oracle.synth_uniform(1, 2, 1)).random_init(1, 1) == 1


def test_degree_stats_hand_case(oracle):  # test_graph.cpp:115-135
    s = line([0.0, 0.0, 0.0])
    g = graph_from(oracle, s, [[(1, 2.0, 0), (2, 1.0, 0)], [(0, 2.0, 0)], []])
    assert g.degree_stats() == {"edges": 3, "max_out": 2, "max_in": 1}
    assert g.degree_stats(cap=1) == {"edges": 2, "max_out": 1, "max_in": 1}


def test_index_bytes_layout_and_crc(oracle):  # graph.cpp:102-126, test_graph.cpp:174-201
    import zlib
    data = oracle.synth_uniform(40, 3, 2)
    g = oracle.OracleGraph(data)
    g.random_init(5, 6)
    b = g.index_bytes()
    assert b[:4] == b"RNND" and int.from_bytes(b[4:8], "little") == 1
    assert int.from_bytes(b[8:16], "little") == 40
    assert int.from_bytes(b[-4:], "little") == zlib.crc32(b[:-4]) & 0xFFFFFFFF
    assert b == g.index_bytes()


# ---------------------------------------------------------- test_search.cpp

def test_search_full_pool_is_exact(oracle):  # test_search.cpp:28-43
    store = oracle.synth_uniform(120, 5, 3)
    queries = oracle.synth_uniform(25, 5, 4)
    gt = oracle.brute_force(store, queries, 3)
    g = oracle.OracleGraph(store)  # edgeless
    for q in range(25):
        ids, _, _, _ = g.search(queries[q], L=120, k=3)
        assert ids.tolist() == gt[q].tolist()


def test_search_hand_case(oracle):  # test_search.cpp:45-64
    store = np.array([[0, 0], [1, 0], [5, 5]], np.float32)
    g = graph_from(oracle, store, [[edge(oracle, store, 0, 1, 0)],
                                   [edge(oracle, store, 1, 0, 0), edge(oracle, store, 1, 2, 0)],
                                   [edge(oracle, store, 2, 1, 0)]])
    q = np.array([0.9, 0.0], np.float32)
    ids, dists, vis, comps = g.search(q, L=3, k=1)
    assert ids.tolist() == [1] and dists[0] == oracle.l2_sq(q, store[1])
    assert vis <= 3 and comps <= 3


def test_search_degree_cap(oracle):  # test_search.cpp:66-90
    s = line([0, 1, 2, 3, 4, 5])
    g = graph_from(oracle, s, [[edge(oracle, s, 0, i, 0) for i in range(1, 6)]] + [[]] * 5)
    ids, _, vis, comps = g.search(np.zeros(1, np.float32), L=6, k=6, K=2, entry_mode=1)
    assert ids.tolist() == [0, 1, 2] and vis == 3 and comps == 3
    ids, _, _, _ = g.search(np.zeros(1, np.float32), L=6, k=6, K=0, entry_mode=1)
    assert len(ids) == 6


def test_search_disconnected_entry(oracle):  # test_search.cpp:92-108
    s = line([0.0, 1.0, 100.0, 101.0])
    g = graph_from(oracle, s, [[edge(oracle, s, 0, 1, 0)], [edge(oracle, s, 1, 0, 0)],
                               [edge(oracle, s, 2, 3, 0)], [edge(oracle, s, 3, 2, 0)]])
    ids, _, _, _ = g.search(np.array([100.5], np.float32), L=2, k=1, entry_mode=1)
    assert ids.tolist() == [1]


# --------------------------------------------------------- test_dataset.cpp

def test_brute_force_hand_cases(oracle):  # test_dataset.cpp:156-183
    base = np.array([[0, 0], [1, 0], [5, 5]], np.float32)
    assert oracle.brute_force(base, np.array([[0.9, 0.0]], np.float32), 2)[0].tolist() == [1, 0]
    dup = np.array([[1, 0], [1, 0], [2, 2]], np.float32)
    assert oracle.brute_force(dup, np.zeros((1, 2), np.float32), 2)[0].tolist() == [0, 1]


def test_brute_force_full_sort(oracle):  # test_dataset.cpp:185-197
    base = oracle.synth_uniform(120, 6, 7)
    qs = oracle.synth_uniform(15, 6, 8)
    gt = oracle.brute_force(base, qs, 9)
    for q in range(15):
        all_ = sorted((oracle.l2_sq(qs[q], base[i]), i) for i in range(120))
        assert gt[q].tolist() == [i for _, i in all_[:9]]


# ------------------------------------------------ committed golden fixtures

def _fixture(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def test_oracle_matches_reference_fixtures(oracle):
    """tests/golden/builds.json was produced by tests/golden/make_golden.py
    from the UNMODIFIED reference (oracle/_ref, rnnd::build threads=4)."""
    fx = _fixture("builds.json")
    assert fx["generator"] == "oracle/_ref rnnd::build threads=4"
    for case in fx["cases"]:
        data = data_for(case)
        assert hashlib.sha256(data.tobytes()).hexdigest() == case["data_sha256"]
        g = oracle.OracleGraph(data)
        rc, pc = g.build(S=case["S"], R=case["R"], T1=case["T1"], T2=case["T2"],
                         seed=case["seed"], order=case["order"])
        assert rc == 0
        assert hashlib.sha256(g.index_bytes()).hexdigest() == case["index_sha256"], case
        assert pc.tolist() == case["per_pass"], case


def test_oracle_matches_reference_live(oracle):
    """When oracle/_ref is built here, compare against it directly."""
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    for (n, d, s) in [(500, 8, 3), (1500, 16, 9)]:
        data = oracle.synth_uniform(n, d, s)
        g = oracle.OracleGraph(data)
        g.build(S=10, R=20, T1=3, T2=4, seed=7)
        r = oracle.RefGraph(data)
        r.build(S=10, R=20, T1=3, T2=4, seed=7, threads=3)
        assert g.index_bytes() == r.index_bytes()
        assert g.export().same_as(r.export())
