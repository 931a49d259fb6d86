"""Debug helper (test infrastructure; imports the oracle): run update passes on the GPU and the oracle side by side and
print the first divergence (counts, then the first differing vertex)."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tests/", 1)[0])
from oracle import oracle as O  # noqa: E402
from paper_2310_20419_b200 import _lib  # noqa: E402
from paper_2310_20419_b200 import rnnd as R  # noqa: E402


def run(data, S, passes=6, seed=7):
    dev = R.Device()
    dev.set_data(R.VectorStore(data))
    dev.check(dev._L.rnndg_random_init(dev.h, S, seed))
    og = O.OracleGraph(data)
    og.random_init(S, seed)
    for p in range(passes):
        before = og.export()
        c = _lib.Counts()
        dev.check(dev._L.rnndg_update_pass(dev.h, C.byref(c)))
        got = [c.removed, c.inserted, c.flag_skips, c.pair_checks]
        want = og.update_pass().tolist()
        g = dev.get_graph()
        a = O.CSR(g.offsets, g.ids, g.dists, g.fresh).canonical()
        b = og.export().canonical()
        same = a.same_as(b)
        print(f"pass {p}: gpu {got} oracle {want} state_equal={same}")
        if got != want or not same:
            for u in range(a.n):
                la = list(zip(a.ids[a.offsets[u]:a.offsets[u + 1]].tolist(),
                              a.fresh[a.offsets[u]:a.offsets[u + 1]].tolist()))
                lb = list(zip(b.ids[b.offsets[u]:b.offsets[u + 1]].tolist(),
                              b.fresh[b.offsets[u]:b.offsets[u + 1]].tolist()))
                if la != lb:
                    bb = before.canonical()
                    print(" vertex", u, "\n  gpu   ", la, "\n  oracle", lb,
                          "\n  before", list(zip(bb.ids[bb.offsets[u]:bb.offsets[u + 1]].tolist(),
                                                 bb.fresh[bb.offsets[u]:bb.offsets[u + 1]].tolist())))
                    break
            return False
    return True


if __name__ == "__main__":
    ok = run(O.synth_uniform(300, 6, 13), 10)
    ok &= run(O.synth_uniform(300, 8, 13), 10)
    ok &= run((np.round(O.synth_uniform(800, 2, 4) * 8) / 8).astype(np.float32), 12)
    print("OK" if ok else "MISMATCH")
