#!/bin/bash
# every BASELINE config on one GPU (bench.py --config X), one JSON line each,
# merged into gpurun_out/configs_1gpu.json
for c in C1-gmm128-20k C2-siftlike-1M C4-deeplike-1M C5-deep10M; do
  timeout 900 python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err || tail -3 gpurun_out/cfg_$c.err
done
python - <<'PY'
import json, glob, os
out = {}
for f in sorted(glob.glob("gpurun_out/cfg_*.json")):
    try:
        d = json.loads(open(f).readline())
    except Exception:
        continue
    keep = {k: d[k] for k in ("value", "unit", "build_seconds", "pair_checks_per_build", "e2e",
                              "roofline", "recall", "stage_seconds", "config", "clocks") if k in d}
    out[os.path.basename(f)[4:-5]] = keep
    print(f, d.get("build_seconds"), d.get("value"), (d.get("recall") or {}).get("L32"))
json.dump(out, open("gpurun_out/configs_1gpu.json", "w"), indent=1)
PY
