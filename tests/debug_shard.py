"""Debug helper: run the sharding protocol with device shards and CPU shards
side by side and report the first step whose owned lists differ."""
import os
import sys

import numpy as np

ROOT = __file__.rsplit("/tests/", 1)[0]
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from shard_cpu import CpuShard  # noqa: E402
from paper_2310_20419_b200 import sharded as SH  # noqa: E402


def lists_dev(e):
    g = e.graph()
    out = {}
    for i, u in enumerate(range(e.v_begin, e.v_end)):
        a, b = int(g.offsets[i]), int(g.offsets[i + 1])
        out[u] = sorted((int(g.ids[j]), float(g.dists[j]), int(g.fresh[j])) for j in range(a, b))
    return out


def lists_cpu(e):
    return {u: sorted((i, float(np.float32(d)), f) for i, d, f in l) for u, l in e.lists.items()}


def compare(tag, devs, cpus):
    for d, c in zip(devs, cpus):
        ld, lc = lists_dev(d), lists_cpu(c)
        for u in ld:
            if ld[u] != lc[u]:
                print("MISMATCH after", tag, "vertex", u)
                print("  dev", ld[u][:12])
                print("  cpu", lc[u][:12])
                return False
    print("ok", tag)
    return True


def main(n=600, world=2, S=8, R=6, order=0):
    from oracle import oracle as O
    data = O.synth_uniform(n, 5, 11)
    b = SH.ownership_bounds(n, world)
    devs = [SH.DeviceShard(data, b[r], b[r + 1]) for r in range(world)]
    cpus = [CpuShard(data, b[r], b[r + 1]) for r in range(world)]
    T = SH.LoopbackTransport()
    for e in devs + cpus:
        e.random_init(S, 5)
    if not compare("init", devs, cpus):
        return

    def both(fn, tag):
        for group in (devs, cpus):
            fn(group)
        return compare(tag, devs, cpus)

    def exch(group, kind, R_=0):
        recvs = T.exchange([e.export(b) for e in group])
        for e, (d, k) in zip(group, recvs):
            e.import_(kind, d, k, R_)

    for t in range(3):
        for group in (devs, cpus):
            pc = [e.scan() for e in group]
        if not both(lambda g: exch(g, SH.X_PENDING), f"apply {t}"):
            return
    for g in (devs, cpus):
        for e in g:
            e.stage(SH.X_PROPOSAL)
    if not both(lambda g: exch(g, SH.X_PROPOSAL), "proposals"):
        return
    if not both(lambda g: [e.out_prune(R) for e in g], "out_prune"):
        return
    for g in (devs, cpus):
        for e in g:
            e.stage(SH.X_INEDGE)
    for g in (devs, cpus):
        recvs = T.exchange([e.export(b) for e in g])
        for e, (d, k) in zip(g, recvs):
            e.import_(SH.X_INEDGE, d, k, R)
    print("staged deletions dev", [e._nstaged for e in devs], "cpu", [len(e.staged) for e in cpus])
    rd = T.exchange([e.export(b) for e in devs])
    rc = T.exchange([e.export(b) for e in cpus])
    for r in range(world):
        dd = sorted(zip(rd[r][0].cpu().tolist(), rd[r][1].cpu().numpy().view(np.uint64).tolist()))
        cc = sorted(zip(rc[r][0].tolist(), rc[r][1].numpy().view(np.uint64).tolist()))
        print("rank", r, "deletion records equal:", dd == cc, len(dd), len(cc))
        if dd != cc:
            print(" dev-only", sorted(set(dd) - set(cc))[:5], " cpu-only", sorted(set(cc) - set(dd))[:5])
    for e, (d, k) in zip(devs, rd):
        e.import_(SH.X_DELETE, d, k, R)
    for e, (d, k) in zip(cpus, rc):
        e.import_(SH.X_DELETE, d, k, R)
    compare("deletions", devs, cpus)


if __name__ == "__main__":
    main()
