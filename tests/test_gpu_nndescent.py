"""NN-Descent baseline on the GPU (nndescent.cpp).

The device runs the canonical deferred join that oracle/rnnd_oracle.c
restates (ro_nnd_pass): pools after init, after every pass (ids, dists,
flags, new-entry counts) and the finalized graph are bit-identical to it.
The init is the reference's own (pools equal rnnd::NnDescent::init with
threads = 1); the join differs from the reference's order-dependent
lock-based one, so the final graph is compared with the reference through
recall, as its own convergence test does (test_nndescent.cpp)."""
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

HAVE_REF = os.path.exists(O.REF_SO)


@pytest.fixture(scope="module")
def R():
    from paper_2310_20419_b200 import rnnd
    return rnnd


def pools_of(nnd):
    return [[(e.id, np.float32(e.dist).view(np.uint32).item(), int(e.fresh)) for e in l]
            for l in nnd.pools()]


def oracle_pools(og):
    c = og.export()
    return [[(int(c.ids[j]), np.float32(c.dists[j]).view(np.uint32).item(), int(c.fresh[j]))
             for j in range(int(c.offsets[u]), int(c.offsets[u + 1]))] for u in range(c.n)]


CASES = [  # (name, data, K, sample, pool)
    ("uniform", lambda: O.synth_uniform(300, 6, 5), 8, 6, 0),
    ("gist-like", lambda: __import__("datagen").rows(3, 3, 0, 400), 10, 10, 30),
    ("grid-ties", lambda: np.stack(np.meshgrid(np.arange(12), np.arange(12)), -1).reshape(-1, 2).astype(np.float32), 6, 8, 0),
    ("sample>=n", lambda: O.synth_uniform(12, 3, 2), 4, 50, 0),
]


@pytest.mark.parametrize("name,make,K,sample,pool", CASES, ids=[c[0] for c in CASES])
def test_pass_by_pass_matches_oracle(R, name, make, K, sample, pool):
    data = np.ascontiguousarray(make(), np.float32)
    cap = max(pool if pool else 2 * K, K)
    p = R.NnDescentParams(K=K, sample=sample, iters=4, pool=pool, seed=7)
    nnd = R.NnDescent(R.VectorStore(data), p)
    nnd.init()
    og = O.OracleGraph(data)
    assert og.nnd_init(K, sample, 4, pool, 7) == 0
    assert pools_of(nnd) == oracle_pools(og)
    for _ in range(4):
        got = nnd.join_pass()
        want = og.nnd_pass(sample, cap)
        assert got == want
        assert pools_of(nnd) == oracle_pools(og)
    g = nnd.finalize()
    assert R.index_bytes(g) == og.nnd_finalize(K).index_bytes()


def test_many_join_chunks(R):
    """Force ~40 join chunks per pass (RNNDG_NND_CHUNK is read once per
    process, so this runs in a child process)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r); import numpy as np\n"
        "from oracle import oracle as O\n"
        "from paper_2310_20419_b200 import rnnd as R\n"
        "x = O.synth_uniform(1500, 5, 3)\n"
        "g = R.build_nndescent(R.VectorStore(x), R.NnDescentParams(K=10, sample=8, iters=3, seed=4))\n"
        "og = O.OracleGraph(x); og.nnd_init(10, 8, 3, 0, 4)\n"
        "[og.nnd_pass(8, 20) for _ in range(3)]\n"
        "assert R.index_bytes(g) == og.nnd_finalize(10).index_bytes()\n"
        "print('ok')\n" % root)
    env = dict(os.environ, RNNDG_NND_CHUNK="2000")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().endswith("ok")


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_init_pools_equal_reference(R):
    x = O.synth_uniform(200, 7, 13)
    K, sample, pool = 8, 6, 0
    (rc, rid, rd), _ = O.ref_nndescent(x, K, sample, 1, pool, seed=9)
    nnd = R.NnDescent(R.VectorStore(x), R.NnDescentParams(K=K, sample=sample, pool=pool, seed=9))
    nnd.init()
    pools = nnd.pools()
    for u in range(200):
        assert len(pools[u]) == int(rc[u])
        assert [e.id for e in pools[u]] == rid[u, :rc[u]].tolist()
        assert all(np.float32(e.dist) == rd[u, j] for j, e in enumerate(pools[u]))
        assert all(e.fresh for e in pools[u])


def test_pool_invariants_and_finalize(R):  # test_nndescent.cpp:69-111
    x = O.synth_uniform(80, 4, 3)
    nnd = R.NnDescent(R.VectorStore(x), R.NnDescentParams(K=6, sample=4, pool=10))
    nnd.init()
    for _ in range(4):
        nnd.join_pass()
    pools = nnd.pools()
    for u, pool in enumerate(pools):
        assert len(pool) <= 10
        ids = [e.id for e in pool]
        assert u not in ids and len(set(ids)) == len(ids)
        assert all((a.dist, a.id) < (b.dist, b.id) for a, b in zip(pool, pool[1:]))
    g = nnd.finalize()
    for u in range(80):
        l = g.list(u)
        assert [e.id for e in l] == [e.id for e in pools[u][:6]]
        assert not any(e.fresh for e in l)


def recall10(g, x):
    gt = O.brute_force(x, x, 11)
    hit = tot = 0
    for u in range(x.shape[0]):
        truth = [i for i in gt[u] if i != u][:10]
        tot += len(truth)
        hit += len(set(truth) & {e.id for e in g.list(u)})
    return hit / tot


def test_converges_like_reference_test(R):  # test_nndescent.cpp:113-134
    x = O.synth_uniform(500, 8, 77)
    g = R.build_nndescent(R.VectorStore(x), R.NnDescentParams(K=10, sample=10, iters=10,
                                                             pool=60))
    assert recall10(g, x) >= 0.90


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_recall_not_below_reference(R):
    import datagen
    x = datagen.rows(1, 0, 0, 4000)  # C1 prefix, d = 128
    p = R.NnDescentParams(K=10, sample=10, iters=6, pool=30, seed=42)
    g = R.build_nndescent(R.VectorStore(x), p)
    _, rg = O.ref_nndescent(x, 10, 10, 6, 30, seed=42)
    gt = O.brute_force(x, x, 11)
    hit_g = hit_r = tot = 0
    for u in range(x.shape[0]):
        truth = set([i for i in gt[u] if i != u][:10])
        tot += len(truth)
        hit_g += len(truth & {e.id for e in g.list(u)})
        hit_r += len(truth & set(rg.ids[int(rg.offsets[u]):int(rg.offsets[u + 1])].tolist()))
    assert hit_g / tot >= hit_r / tot - 0.005


def test_deterministic_and_validates(R):  # test_nndescent.cpp:136-160
    x = O.synth_uniform(150, 4, 11)
    p = R.NnDescentParams(K=8, sample=6, iters=4)
    a = R.build_nndescent(R.VectorStore(x), p)
    b = R.build_nndescent(R.VectorStore(x), p)
    assert R.index_bytes(a) == R.index_bytes(b)
    small = R.VectorStore(O.synth_uniform(10, 3, 1))
    for kw, msg in ((dict(K=0), "K out of"), (dict(K=10), "K out of"),
                    (dict(K=3, sample=0), "sample must be"), (dict(K=3, iters=0), "iters must be")):
        with pytest.raises(R.ParamError, match=msg):
            R.build_nndescent(small, R.NnDescentParams(**kw))
    with pytest.raises(R.ParamError, match="need at least 2"):
        R.build_nndescent(R.VectorStore(O.synth_uniform(1, 3, 1)), R.NnDescentParams(K=1))
