"""Time the parts of the e2e leg of bench.py: H2D (set_data), build, D2H (get_graph)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2310_20419_b200 import rnnd as R, datagen

cfg = datagen.CONFIGS["C3-gistlike-1M"]
data = datagen.rows(cfg.cfg, cfg.seed, 0, cfg.n)
pinned = torch.empty(data.shape, dtype=torch.float32, pin_memory=True)
pinned.numpy()[:] = data
ps = R.VectorStore(pinned.numpy())
dev = R.Device()
params = R.BuildParams(S=20, R=96, T1=4, T2=15)
for it in range(3):
    t0 = time.perf_counter(); dev.set_data(ps); t1 = time.perf_counter()
    st = R.BuildStats(); R.build(ps, params, st, device=dev); t2 = time.perf_counter()
    g = dev.get_graph(); t3 = time.perf_counter()
    print(f"h2d {t1-t0:.4f}s ({data.nbytes/(t1-t0)/1e9:.1f} GB/s) build {t2-t1:.4f}s (stats {st.seconds:.4f}) d2h {t3-t2:.4f}s ({len(g.ids)} edges)")
