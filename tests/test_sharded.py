"""Sharded build: the vertex-ownership protocol gives the same
graph and the same per-pass counters as the unsharded build.

CPU (gloo / loopback) runs use tests/shard_cpu.py; the GPU run uses the real
device shards (rnndg_set_partition + rnndg_shard_*) with the in-process
loopback transport on one device.
"""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2310_20419_b200 import sharded as SH

PARAMS = dict(S=8, R=10, T1=3, T2=3, seed=5)


def reference_graph(data, order=0):
    g = O.OracleGraph(data)
    rc, pc = g.build(order=order, **PARAMS)
    assert rc == 0
    c = g.export()
    lists = {u: [(int(c.ids[j]), float(c.dists[j])) for j in range(int(c.offsets[u]), int(c.offsets[u + 1]))]
             for u in range(c.n)}
    return lists, pc


def shard_lists(engines):
    out = {}
    for e in engines:
        for u, l in e.sorted_lists().items():
            out[u] = [(i, d) for i, d, _ in l]
    return out


def test_ownership_bounds():
    assert SH.ownership_bounds(10, 3) == [0, 3, 6, 10]
    assert SH.ownership_bounds(2, 4) == [0, 0, 1, 1, 2]


@pytest.mark.parametrize("world,order", [(1, 0), (2, 0), (3, 1), (4, 0)])
def test_loopback_cpu_matches_unsharded(world, order):
    from shard_cpu import CpuShard
    data = O.synth_uniform(240, 5, 3)
    b = SH.ownership_bounds(240, world)
    engines = [CpuShard(data, b[r], b[r + 1]) for r in range(world)]
    st = SH.sharded_build(engines, SH.LoopbackTransport(), 240, world, order=order, **PARAMS)
    ref, pc = reference_graph(data, order)
    assert [list(map(int, c)) for c in st.pass_counts] == pc.tolist()
    assert shard_lists(engines) == ref


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, data, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from shard_cpu import CpuShard
        n = data.shape[0]
        b = SH.ownership_bounds(n, world)
        eng = CpuShard(data, b[rank], b[rank + 1])
        st = SH.sharded_build([eng], SH.TorchDistTransport(), n, world, **PARAMS)
        parts = [None] * world
        dist.all_gather_object(parts, shard_lists([eng]))
        if rank == 0:
            merged = {}
            for p in parts:
                merged.update(p)
            q.put(([list(map(int, c)) for c in st.pass_counts], merged))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_two_ranks_match_unsharded(world):
    import sys
    import torch.multiprocessing as mp
    here = os.path.dirname(os.path.abspath(__file__))
    root = os.path.dirname(here)
    for p in (here, root):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ["PYTHONPATH"] = os.pathsep.join([here, root, os.environ.get("PYTHONPATH", "")])
    data = O.synth_uniform(200, 4, 9)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, data, q)) for r in range(world)]
    for p in procs:
        p.start()
    counts, merged = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref, pc = reference_graph(data)
    assert counts == pc.tolist()
    assert merged == ref


@pytest.mark.gpu
@pytest.mark.parametrize("world,order", [(2, 0), (3, 1)])
def test_device_shards_match_single_device(world, order):
    """Real device shards (rnndg_set_partition + rnndg_shard_*) on one GPU,
    records moved in-process: identical graph and counters to the
    single-context build."""
    import datagen
    from paper_2310_20419_b200 import rnnd as R
    data = datagen.rows(4, 4, 0, 3000)  # C4 (Deep-like) generator prefix
    b = SH.ownership_bounds(3000, world)
    engines = [SH.DeviceShard(data, b[r], b[r + 1]) for r in range(world)]
    p = dict(S=20, R=24, T1=3, T2=5, seed=42)
    st = SH.sharded_build(engines, SH.LoopbackTransport(), 3000, world, order=order, **p)
    single = R.BuildStats()
    g = R.build(R.VectorStore(data), R.BuildParams(S=20, R=24, T1=3, T2=5, seed=42,
                                                   prune_order=R.PruneOrder(order)), single)
    assert [list(map(int, c)) for c in st.pass_counts] == \
        [[c.removed, c.inserted, c.flag_skips, c.pair_checks] for c in single.pass_counts]
    ref = g.csr
    for e, lo, hi in zip(engines, b[:-1], b[1:]):
        part = e.graph()
        roff = ref.offsets[lo:hi + 1] - ref.offsets[lo]
        assert np.array_equal(part.offsets, roff)
        assert np.array_equal(part.ids, ref.ids[int(ref.offsets[lo]):int(ref.offsets[hi])])
        assert np.array_equal(part.dists.view(np.uint32),
                              ref.dists[int(ref.offsets[lo]):int(ref.offsets[hi])].view(np.uint32))


@pytest.mark.gpu
def test_nccl_transport_matches_single_device():
    """The bench's N > 1 path end to end at one rank: TorchDistTransport over
    NCCL, C5 generator prefix (1M rows), identical to the single-context
    build (tests/nccl_case.py)."""
    import random
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    port = random.randint(29600, 29900)
    r = subprocess.run([sys.executable, os.path.join(here, "nccl_case.py"), "1000000", str(port)],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
