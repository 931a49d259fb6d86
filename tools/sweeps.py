"""Recall / QPS sweeps with the paper's out-degree (K) ablation on the B200
(the reference's sweep_search / sweep_build /
report_aod_table, eval.cpp:93-152), through paper_2310_20419_b200.evaluate.

usage: python tools/sweeps.py CONFIG [CONFIG ...]   (C3-gistlike-1M, ...)
writes gpurun_out/sweep_<config>.csv (eval.cpp CSV) and .json (AOD table,
(T1, T2) build sweep, timings)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
from paper_2310_20419_b200 import evaluate as E  # noqa: E402
from paper_2310_20419_b200 import rnnd as R  # noqa: E402

LS = [16, 24, 32, 48, 64, 96, 128]
KS = [16, 32, 48, 64, 96, 0]  # 0 = uncapped
T_PAIRS = [(1, 60), (2, 30), (4, 15), (6, 10)]


def main(name):
    cfg = datagen.CONFIGS[name]
    nq = {"C1-gmm-20k": 1000, "C3-gistlike-1M": 1000}.get(name, 10000)
    base = R.VectorStore(datagen.rows(cfg.cfg, cfg.seed, 0, cfg.n))
    queries = R.VectorStore(datagen.rows(cfg.cfg, cfg.seed, cfg.n, nq))
    dev = R.Device()
    dev.set_data(base)
    t = time.perf_counter()
    gt = R.brute_force_gt(base, queries, 1, device=dev)
    gt_s = time.perf_counter() - t
    st = R.BuildStats()
    g = R.build(base, R.BuildParams(), st, device=dev)
    ctx = E.RowContext(name, "rnn-descent", 20, 96, 4, 15, st.seconds)
    rows = E.sweep_search(g, base, queries, gt, LS, KS, E.SweepOptions(k=1, reps=3), ctx)
    aod = E.report_aod_table(g, [16, 32, 48, 64, 96])
    brows = []
    if cfg.n <= 1_000_000:
        brows = E.sweep_build(base, queries, gt, T_PAIRS, R.BuildParams(),
                              R.SearchParams(L=64, K=0, k=1), E.SweepOptions(k=1, reps=3), name)
    out = os.path.join(ROOT, "gpurun_out", f"sweep_{name}")
    E.write_csv(rows + brows, out + ".csv")
    with open(out + ".json", "w") as f:
        json.dump({"config": name, "rows": cfg.n, "queries": nq, "build_seconds": st.seconds,
                   "gt_seconds": gt_s, "aod_by_cap": aod,
                   "build_sweep": [{"T1": r.T1, "T2": r.T2, "build_s": r.build_seconds,
                                    "recall@1_L64": r.recall_at_1, "qps": r.qps}
                                   for r in brows]}, f, indent=1)
    best = max(rows, key=lambda r: (r.recall_at_1, r.qps))
    print(name, f"build {st.seconds:.3f} s", f"best recall@1 {best.recall_at_1:.4f}",
          f"pareto points {sum(r.pareto for r in rows)}")


if __name__ == "__main__":
    for name in sys.argv[1:]:
        main(name)
