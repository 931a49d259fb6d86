"""One C3 1M build through the C ABI (profiling driver: ncu / sanitizer runs).

usage: python tools/prof_build.py [config] [rows]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from paper_2310_20419_b200 import rnnd as R  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3-gistlike-1M"
cfg = datagen.CONFIGS[name]
n = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n
data = datagen.rows(cfg.cfg, cfg.seed, 0, n)
store = R.VectorStore(data)
dev = R.Device()
dev.set_data(store)
st = R.BuildStats()
g = R.build(store, R.BuildParams(), st, device=dev)
print(f"build {st.seconds:.4f} s, scan {st.scan_seconds:.4f} s, checks {st.edits.pair_checks}")
