"""Generate tests/golden/* from the UNMODIFIED reference (oracle/_ref).

Run here (needs /root/reference to build oracle/_ref):
    make -C oracle all ref && python tests/golden/make_golden.py

builds.json  - rnnd::build(threads=4) on small seeded stores: sha256 of the
               serialized RNND index, total EditCounts and per-pass counts.
search.npz   - rnnd::batch_search / brute_force_gt on one of those graphs.
Inputs are regenerated at test time (oracle synth_uniform = the reference's
synth_uniform, or the seeded datagen package, whose bytes are hashed too).
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
import datagen  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_data import data_for  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


CASES = [
    dict(kind="uniform", n=300, d=6, data_seed=13, S=10, R=16, T1=2, T2=4, seed=5, order=0),
    dict(kind="uniform", n=1000, d=5, data_seed=21, S=8, R=12, T1=3, T2=3, seed=9, order=1),
    dict(kind="uniform", n=2000, d=16, data_seed=3, S=20, R=96, T1=4, T2=15, seed=42, order=0),
    dict(kind="grid", n=800, d=2, data_seed=4, S=12, R=10, T1=3, T2=5, seed=1, order=0),
    dict(kind="grid", n=600, d=3, data_seed=5, S=6, R=5, T1=3, T2=4, seed=2, order=1),
    dict(kind="cfg", cfg=1, n=3000, d=128, data_seed=0, S=20, R=96, T1=4, T2=15, seed=42, order=0),
    dict(kind="cfg", cfg=2, n=3000, d=128, data_seed=2, S=20, R=96, T1=4, T2=15, seed=42, order=0),
    dict(kind="cfg", cfg=3, n=1500, d=960, data_seed=3, S=20, R=96, T1=4, T2=15, seed=42, order=0),
    dict(kind="cfg", cfg=4, n=3000, d=96, data_seed=4, S=20, R=96, T1=4, T2=15, seed=42, order=0),
]


def main():
    out = {"generator": "oracle/_ref rnnd::build threads=4", "cases": []}
    graphs = {}
    for case in CASES:
        data = data_for(case)
        r = O.RefGraph(data)
        r.random_init(case["S"], case["seed"])
        per_pass = []
        for t1 in range(1, case["T1"] + 1):
            for _ in range(case["T2"]):
                per_pass.append(r.update_pass(threads=4).tolist())
            if t1 != case["T1"]:
                assert r.add_reverse_edges(case["R"], threads=4, order=case["order"]) == 0
        # the same thing through rnnd::build itself
        rb = O.RefGraph(data)
        rc, st = rb.build(S=case["S"], R=case["R"], T1=case["T1"], T2=case["T2"],
                          seed=case["seed"], threads=4, order=case["order"])
        assert rc == 0
        idx = rb.index_bytes()
        c = dict(case)
        c["data_sha256"] = hashlib.sha256(data.tobytes()).hexdigest()
        c["index_sha256"] = hashlib.sha256(idx).hexdigest()
        c["edits"] = [int(st[3]), int(st[4]), int(st[5]), int(st[6])]
        c["per_pass"] = per_pass
        assert np.array(per_pass).sum(0).tolist() == c["edits"]
        c["edges"] = int(rb.export().offsets[-1])
        out["cases"].append(c)
        graphs[len(out["cases"]) - 1] = (rb, data)
        print(case["kind"], case.get("cfg"), case["n"], case["d"], c["edits"], c["edges"])
    with open(os.path.join(HERE, "builds.json"), "w") as f:
        json.dump(out, f, indent=1)

    # search goldens on the C1-prefix graph (case 5)
    rb, data = graphs[5]
    q = datagen.rows(1, 0, 3000, 200)
    arrays = {"queries_sha256": np.frombuffer(
        hashlib.sha256(q.tobytes()).digest(), np.uint8)}
    for L, K in [(10, 0), (32, 0), (64, 16), (16, 4)]:
        ids, dists, vis, comps, _ = rb.batch_search(q, L=L, K=K, k=10, seed=42, threads=4)
        arrays[f"ids_L{L}_K{K}"] = ids
        arrays[f"dists_L{L}_K{K}"] = dists
        arrays[f"visited_L{L}_K{K}"] = vis
        arrays[f"comps_L{L}_K{K}"] = comps
    arrays["gt10"] = O.ref_brute_force(data, q, 10, threads=4)
    np.savez_compressed(os.path.join(HERE, "search.npz"), **arrays)
    print("wrote builds.json, search.npz")


if __name__ == "__main__":
    main()
