"""Full-size goldens from the UNMODIFIED reference (oracle/_ref): BASELINE.json
configs C2/C3/C4 at 1,000,000 rows, and a 1,000,000-row prefix of C5.

Run here (needs oracle/_ref, ~1 h on 8 cores for all four):
    make -C oracle all ref && python tests/golden/make_golden_1m.py [C3 C2 C4 C5p]

For each config it records, into tests/golden/builds_1m.json:
  * data_sha256          sha256 of the generated base rows (datagen bytes)
  * index_sha256, edges  of rnnd::build(S=20,R=96,T1=4,T2=15,seed=42,
                         threads=nproc) -> save_index bytes (graph.cpp:102-126)
  * ref_seconds          BuildStats.seconds of that build (builder.cpp:260-286),
                         with threads, CPU model and date: the same-config CPU time
  * per_pass             EditCounts of each of the 60 passes, from the same
                         schedule driven through update_neighbors /
                         add_reverse_edges (threads=nproc); the resulting graph
                         is checked to equal rnnd::build's list for list
  * recall               rnnd::batch_search (K=0, k=10, seed 42) at L=16/32/64
                         on the held-out queries against brute_force_gt (k=10):
                         recall@1 by the reference's tie-tolerant rule
                         (eval.cpp:57-76), recall@10 = |top10 & gt10| / 10
  * aod, max_out         mean / max out-degree (degree_stats, graph.cpp:76-100)
and into tests/golden/gt_<cfg>.npz the brute-force top-10 ids (the GPU tests
reuse them as the recall ground truth and as a brute-force parity check).
"""
import datetime
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
import datagen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "builds_1m.json")

# name -> (datagen config, rows, queries)
TARGETS = {
    "C3": (datagen.C3, 1_000_000, 1_000),
    "C2": (datagen.C2, 1_000_000, 10_000),
    "C4": (datagen.C4, 1_000_000, 10_000),
    "C5p": (datagen.C5, 1_000_000, 10_000),  # 1M-row prefix of the 10M config
}
S, R, T1, T2, SEED = 20, 96, 4, 15, 42
LS = (16, 32, 64)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def recall_at_1(data, q, ids, gt):
    """eval.cpp:57-76: hit if ids[0]==gt[0] or l2(q, x[ids[0]]) == l2(q, x[gt[0]])."""
    hit = 0
    for i in range(q.shape[0]):
        a, b = int(ids[i, 0]), int(gt[i, 0])
        if a == b or np.float32(O.l2_sq(q[i], data[a])) == np.float32(O.l2_sq(q[i], data[b])):
            hit += 1
    return hit / q.shape[0]


def recall_at_10(ids, gt):
    return float(np.mean([len(set(ids[i, :10].tolist()) & set(gt[i, :10].tolist())) / 10.0
                          for i in range(ids.shape[0])]))


def run(name: str, threads: int) -> dict:
    cfg, n, nq = TARGETS[name]
    t0 = time.time()
    data = datagen.rows(cfg.cfg, cfg.seed, 0, n)
    q = datagen.rows(cfg.cfg, cfg.seed, cfg.n, nq)
    print(f"[{name}] data {data.shape} in {time.time() - t0:.1f}s", flush=True)

    rb = O.RefGraph(data)
    rc, st = rb.build(S=S, R=R, T1=T1, T2=T2, seed=SEED, threads=threads, order=0)
    assert rc == 0
    idx = rb.index_bytes()
    print(f"[{name}] rnnd::build {st[0]:.1f}s edges {int(rb.export().offsets[-1])}", flush=True)
    built = rb.export()

    # same schedule pass by pass, for the per-pass counters
    rl = O.RefGraph(data)
    assert rl.random_init(S, SEED) == 0
    per_pass = []
    for t1 in range(1, T1 + 1):
        for _ in range(T2):
            per_pass.append([int(x) for x in rl.update_pass(threads=threads)])
        if t1 != T1:
            assert rl.add_reverse_edges(R, threads=threads, order=0) == 0
    looped = rl.export()
    assert looped.same_as(built), "pass-by-pass schedule differs from rnnd::build"
    del rl
    tot = np.array(per_pass, dtype=np.uint64).sum(0).tolist()
    assert tot == [int(st[3]), int(st[4]), int(st[5]), int(st[6])]
    print(f"[{name}] per-pass ok, totals {tot}", flush=True)

    t1_ = time.time()
    gt = O.ref_brute_force(data, q, 10, threads=threads)
    print(f"[{name}] brute force {time.time() - t1_:.1f}s", flush=True)
    recall = {}
    for L in LS:
        ids, dists, vis, comps, wall = rb.batch_search(q, L=L, K=0, k=10, seed=42,
                                                       threads=threads)
        recall[f"L{L}"] = {"recall@1": recall_at_1(data, q, ids, gt),
                           "recall@10": recall_at_10(ids, gt),
                           "ids_sha256": hashlib.sha256(ids.tobytes()).hexdigest(),
                           "qps": nq / wall if wall > 0 else None}
    lens = np.diff(built.offsets.astype(np.int64))
    np.savez_compressed(os.path.join(HERE, f"gt_{name}.npz"), gt10=gt)
    return {
        "config": cfg.name, "rows": n, "dim": int(data.shape[1]), "queries": nq,
        "datagen": {"cfg": cfg.cfg, "seed": cfg.seed, "query_row0": cfg.n},
        "S": S, "R": R, "T1": T1, "T2": T2, "seed": SEED, "prune_order": "kOutThenIn",
        "data_sha256": hashlib.sha256(data.tobytes()).hexdigest(),
        "queries_sha256": hashlib.sha256(q.tobytes()).hexdigest(),
        "index_sha256": hashlib.sha256(idx).hexdigest(),
        "index_bytes": len(idx),
        "edges": int(built.offsets[-1]),
        "edits": tot,
        "per_pass": per_pass,
        "ref_seconds": float(st[0]),
        "ref_threads": threads,
        "cpu_model": cpu_model(),
        "date": datetime.datetime.utcnow().strftime("%Y-%m-%dT%H:%M:%SZ"),
        "recall": recall,
        "aod": float(lens.mean()),
        "max_out": int(lens.max()),
    }


def main():
    names = sys.argv[1:] or list(TARGETS)
    threads = O.ref_lib().ref_max_threads()
    out = {"generator": "oracle/_ref rnnd::build (unmodified reference)", "configs": {}}
    if os.path.exists(OUT):
        with open(OUT) as f:
            out = json.load(f)
    for name in names:
        out["configs"][name] = run(name, threads)
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1)
        print(f"[{name}] written", flush=True)


if __name__ == "__main__":
    main()
