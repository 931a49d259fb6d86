"""every BASELINE config on one B200 next to
the UNMODIFIED reference (oracle/_ref, rnnd::build(threads = all host cores),
BuildStats.seconds) on the box's host cores -- the full config, the same rows.
CPU: one untimed warm-up + median of 3 for C1-C4, one run for C5.  GPU:
bench.py --config X (its own JSON line, CPU leg off).

usage (GPU box, repo root): python tools/side_by_side.py [config ...]
writes gpurun_out/side_by_side.json"""
import datetime
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import datagen  # noqa: E402
from oracle import oracle as O  # noqa: E402

GPU_ONLY = "--gpu-only" in sys.argv  # re-measure the GPU legs, keep the recorded CPU legs
sys.argv = [a for a in sys.argv if a != "--gpu-only"]
names = sys.argv[1:] or ["C1-gmm128-20k", "C2-siftlike-1M", "C3-gistlike-1M", "C4-deeplike-1M",
                         "C5-deep10M"]
out = {"date": datetime.datetime.now(datetime.timezone.utc).isoformat(), "cpu_model": bench.cpu_model(),
       "host_threads": max(len(os.sched_getaffinity(0)), 2), "configs": {}}
path = os.path.join(ROOT, "gpurun_out", "side_by_side.json")
prev = {}
if GPU_ONLY:
    prev = json.load(open(os.path.join(ROOT, "profiles", "r02_side_by_side_all_configs.json")))
    out["cpu_legs_from"] = prev.get("date")
for name in names:
    cfg = datagen.CONFIGS[name]
    rec = {}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", name,
                        "--steps", "3", "--warmup", "1", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=3000)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        rec["gpu"] = {k: d.get(k) for k in ("value", "unit", "build_seconds",
                                            "pair_checks_per_build", "stage_seconds", "roofline",
                                            "e2e", "recall", "parity", "clocks", "gpu_launches")}
    except Exception as e:  # keep going: the CPU leg is still worth having
        rec["gpu"] = {"failed": str(e), "stderr": r.stderr[-500:]}
    if GPU_ONLY:
        rec["cpu_reference"] = prev["configs"][name]["cpu_reference"]
        med, checks = rec["cpu_reference"]["seconds_median"], rec["cpu_reference"]["pair_checks"]
        gb = rec["gpu"].get("build_seconds")
        if gb:
            rec["gpu_over_cpu_build_time"] = med / gb
            rec["pair_checks_equal"] = rec["gpu"].get("pair_checks_per_build") == int(checks)
        out["configs"][name] = rec
        json.dump(out, open(path, "w"), indent=1)
        print(name, json.dumps({"gpu_s": gb, "cpu_s": med,
                                "checks_equal": rec.get("pair_checks_equal")}), flush=True)
        continue
    data = bench.store_rows(cfg, cfg.n)
    runs = 1 if cfg.n > 2_000_000 else 3
    secs, checks = [], None
    for i in range(runs + (1 if runs > 1 else 0)):  # warm-up run for the small configs
        g = O.RefGraph(data)
        rc, st = g.build(threads=out["host_threads"])
        assert rc == 0
        if runs > 1 and i == 0:
            continue
        secs.append(float(st[0]))
        checks = float(st[6])
        del g
    med = statistics.median(secs)
    rec["cpu_reference"] = {"seconds_runs": secs, "seconds_median": med, "pair_checks": checks,
                            "dist_evals_per_s": checks / med, "threads": out["host_threads"],
                            "what": f"rnnd::build(threads={out['host_threads']}) on all "
                                    f"{cfg.n} rows of {name}"}
    gb = rec["gpu"].get("build_seconds")
    if gb:
        rec["gpu_over_cpu_build_time"] = med / gb
        rec["pair_checks_equal"] = rec["gpu"].get("pair_checks_per_build") == int(checks)
    out["configs"][name] = rec
    json.dump(out, open(path, "w"), indent=1)
    print(name, json.dumps({"gpu_s": gb, "cpu_s": med, "checks_equal": rec.get("pair_checks_equal")}),
          flush=True)
