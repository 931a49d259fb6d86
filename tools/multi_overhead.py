"""Overhead of the in-process sharded protocol (csrc/multi.cu) on ONE GPU:
a C3 1M build through rnndg_sharded_* with 1 shard (and 2 shards sharing the
GPU -- correctness of the concurrent host threads at scale, not a scaling
number), fused exchange (rnndg_shard_push) vs sorted export + peer copies,
against the single-context rnndg_build.

usage: python tools/multi_overhead.py [config] [rows]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from paper_2310_20419_b200 import rnnd as R  # noqa: E402
from paper_2310_20419_b200.sharded import MultiDevice  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3-gistlike-1M"
cfg = datagen.CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
data = datagen.rows(cfg.cfg, cfg.seed, 0, n)
out = {"config": name, "rows": n}
store = R.VectorStore(data)
dev = R.Device()
dev.set_data(store)
for _ in range(2):
    st = R.BuildStats()
    g = R.build(store, R.BuildParams(), st, device=dev)
out["single_context_s"] = st.seconds
ref = [[c.removed, c.inserted, c.flag_skips, c.pair_checks] for c in st.pass_counts]
del g, dev
for shards in (1, 2):
    for mode in ("push", "copy"):
        os.environ["RNNDG_MULTI_EXCHANGE"] = mode
        md = MultiDevice([0] * shards)
        md.set_data(data)
        best = None
        for _ in range(2):
            t0 = time.perf_counter()
            st, counts = md.build()
            dt = time.perf_counter() - t0
            best = dt if best is None or dt < best else best
        assert counts == ref, "per-pass counts differ from the single-context build"
        out[f"{shards}shard_{mode}_s"] = best
        md.close()
print(json.dumps(out))
