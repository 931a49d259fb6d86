"""The oracle's NN-Descent (oracle/rnnd_oracle.c ro_nnd_*) against the
reference: init pools identical to rnnd::NnDescent::init (threads = 1), the
deferred join keeps the reference's pool invariants and converges at least
as well as the reference's own join on its convergence case
(test_nndescent.cpp:113-134)."""
import os

import numpy as np
import pytest

from oracle import oracle as O

HAVE_REF = os.path.exists(O.REF_SO)


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("n,d,K,sample,pool", [(200, 7, 8, 6, 0), (60, 3, 5, 64, 12)])
def test_init_equals_reference(n, d, K, sample, pool):
    x = O.synth_uniform(n, d, 13)
    (rc, rid, rd), _ = O.ref_nndescent(x, K, sample, 1, pool, seed=9)
    og = O.OracleGraph(x)
    assert og.nnd_init(K, sample, 1, pool, 9) == 0
    c = og.export()
    for u in range(n):
        a, b = int(c.offsets[u]), int(c.offsets[u + 1])
        assert b - a == int(rc[u])
        assert c.ids[a:b].tolist() == rid[u, :rc[u]].tolist()
        assert c.dists[a:b].view(np.uint32).tolist() == rd[u, :rc[u]].view(np.uint32).tolist()
        assert all(c.fresh[a:b])


def test_invariants_and_no_join_without_fresh():
    x = O.synth_uniform(80, 4, 3)
    og = O.OracleGraph(x)
    assert og.nnd_init(6, 4, 4, 10, 42) == 0
    for _ in range(12):
        og.nnd_pass(4, 10)
    c = og.export()
    for u in range(80):
        a, b = int(c.offsets[u]), int(c.offsets[u + 1])
        ids = c.ids[a:b].tolist()
        assert b - a <= 10 and u not in ids and len(set(ids)) == len(ids)
        keys = list(zip(c.dists[a:b].tolist(), ids))
        assert keys == sorted(keys)
    # converged: once no entry is fresh, a pass joins nothing (test_nndescent.cpp:49-67)
    while og.nnd_pass(4, 10):
        pass
    assert og.nnd_pass(4, 10) == 0


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")
def test_convergence_at_least_reference():
    x = O.synth_uniform(500, 8, 77)
    og = O.OracleGraph(x)
    assert og.nnd_init(10, 10, 10, 60, 42) == 0
    for _ in range(10):
        og.nnd_pass(10, 60)
    f = og.nnd_finalize(10).export()
    _, rg = O.ref_nndescent(x, 10, 10, 10, 60)
    gt = O.brute_force(x, x, 11)
    hit = hit_r = tot = 0
    for u in range(500):
        t = set([i for i in gt[u] if i != u][:10])
        tot += len(t)
        hit += len(t & set(f.ids[int(f.offsets[u]):int(f.offsets[u + 1])].tolist()))
        hit_r += len(t & set(rg.ids[int(rg.offsets[u]):int(rg.offsets[u + 1])].tolist()))
    assert hit / tot >= 0.90
    assert hit / tot >= hit_r / tot
