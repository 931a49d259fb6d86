"""Parity of the distance stage under one setting of the RNNDG_* schedule
knobs (read once per process, so tests/test_gpu_knobs.py starts this script
per setting).  Two cases, each against the CPU oracle (oracle/rnnd_oracle.c,
pinned to the reference):

  passes  d = 67 (a d % 4 tail; RNNDG_CASE_D overrides it: d = 96 / 128 take
          the shared-memory walk of rowwalk.cu), imported lists of every size class -- Gram
          tiles of 16/32/64/128 rows, short lists up to 384, hubs -- then
          update passes, a reverse phase and more passes; the whole graph and
          every EditCounts compared after each step
  build   a 2,500-row prefix of the C3 generator (d = 960), a full build
          (S=20 R=96 T1=2 T2=4): index bytes and per-pass counts

Exits 0 on parity."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def case_passes() -> int:
    from oracle import oracle
    from oracle.oracle import CSR
    from paper_2310_20419_b200 import _lib, rnnd as R

    n, d = 4000, int(os.environ.get("RNNDG_CASE_D", "67"))
    data = oracle.synth_uniform(n, d, 5)
    rng = np.random.default_rng(3)
    sizes = [2, 9, 16, 17, 31, 32, 33, 63, 64, 65, 100, 127, 128, 129, 200, 383, 384, 385, 700,
             1500]
    lists = []
    for u in range(n):
        m = sizes[u % len(sizes)] if u < 400 else 5 + u % 40
        lists.append(rng.choice(np.delete(np.arange(n), u), m, replace=False).astype(np.uint32))
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(x) for x in lists])
    ids = np.concatenate(lists)
    owner = np.repeat(np.arange(n), [len(x) for x in lists])
    dists = np.array([oracle.l2_sq(data[u], data[v]) for u, v in zip(owner, ids)], np.float32)
    fresh = (rng.random(len(ids)) < 0.7).astype(np.uint8)
    dev = R.Device()
    dev.set_data(R.VectorStore(data))
    dev.set_graph(R.CSR(off, ids, dists, fresh), True)
    og = oracle.OracleGraph(data)
    og.load(CSR(off, ids, dists, fresh))

    def same(step):
        g = dev.get_graph()
        if not CSR(g.offsets, g.ids, g.dists, g.fresh).same_as(og.export()):
            print("graph differs after", step)
            return False
        return True

    for p in range(6):
        if p == 3:
            dev.check(dev._L.rnndg_reverse(dev.h, 40, 0))
            og.add_reverse_edges(40, 0)
            if not same("reverse"):
                return 1
        c = _lib.Counts()
        dev.check(dev._L.rnndg_update_pass(dev.h, C.byref(c)))
        got = [int(c.removed), int(c.inserted), int(c.flag_skips), int(c.pair_checks)]
        want = og.update_pass().tolist()
        if got != want:
            print("counts differ", p, got, want)
            return 1
        if not same(f"pass {p}"):
            return 1
    return 0


def case_build() -> int:
    import datagen
    from oracle import oracle
    from paper_2310_20419_b200 import rnnd as R

    data = datagen.rows(3, 3, 0, 2500)
    st = R.BuildStats()
    g = R.build(R.VectorStore(data), R.BuildParams(S=20, R=96, T1=2, T2=4), st)
    og = oracle.OracleGraph(data)
    rc, pc = og.build(S=20, R=96, T1=2, T2=4)
    got = [[c.removed, c.inserted, c.flag_skips, c.pair_checks] for c in st.pass_counts]
    if rc != 0 or got != pc.tolist():
        print("pass counts differ", got, pc.tolist())
        return 1
    if R.index_bytes(g) != og.index_bytes():
        print("index bytes differ")
        return 1
    return 0


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "passes"
    rc = case_passes() if which == "passes" else case_build()
    print("ok" if rc == 0 else "FAIL")
    sys.exit(rc)
