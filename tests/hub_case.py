"""Hub-heavy update passes checked against the CPU oracle, run as a script so
that tests/test_gpu_hub_modes.py can start it under different scan settings
(the RNNDG_* knobs are read once per process).  Exits 0 on parity."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(nhubs: int) -> int:
    from oracle import oracle
    from oracle.oracle import CSR
    from paper_2310_20419_b200 import _lib, rnnd as R

    n, d = 6000, 16
    data = oracle.synth_uniform(n, d, 91)
    rng = np.random.default_rng(11)
    lists = []
    for u in range(n):
        if u == 0:
            m = 2500          # a big hub (cluster-cooperative walk)
        elif u <= nhubs:
            m = 300 + (u % 7) * 90  # mid-size hubs, 300 .. 840 entries
        else:
            m = 10 + u % 9
        lists.append(rng.choice(np.delete(np.arange(n), u), m, replace=False).astype(np.uint32))
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in lists])
    ids = np.concatenate(lists)
    owner = np.repeat(np.arange(n), [len(x) for x in lists])
    dists = np.array([oracle.l2_sq(data[u], data[v]) for u, v in zip(owner, ids)], np.float32)
    fresh = (rng.random(len(ids)) < 0.6).astype(np.uint8)
    dev = R.Device()
    dev.set_data(R.VectorStore(data))
    dev.set_graph(R.CSR(off, ids, dists, fresh), True)
    og = oracle.OracleGraph(data)
    og.load(CSR(off, ids, dists, fresh))
    for p in range(3):
        c = _lib.Counts()
        dev.check(dev._L.rnndg_update_pass(dev.h, C.byref(c)))
        got = [int(c.removed), int(c.inserted), int(c.flag_skips), int(c.pair_checks)]
        want = og.update_pass().tolist()
        if got != want:
            print("counts differ", p, got, want)
            return 1
        g = dev.get_graph()
        if not CSR(g.offsets, g.ids, g.dists, g.fresh).same_as(og.export()):
            print("graph differs after pass", p)
            return 1
    print("ok")
    return 0


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]) if len(sys.argv) > 1 else 400))
