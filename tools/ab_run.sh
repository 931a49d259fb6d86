#!/bin/bash
# usage (GPU box, repo root): tools/ab_run.sh TAG "ENV=.. ENV2=.." [TAG2 "ENV.."]...
# one C3 bench (3 timed builds) per variant, traced; summary line per variant
while [ $# -ge 2 ]; do
  tag=$1; envs=$2; shift 2
  env $envs RNNDG_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --no-recall --steps 3 --warmup 3 > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{t}.json").readline())
    print(t, "build_s %.4f scan %.4f frac %.4f" % (d["build_seconds"], d["stage_seconds"]["scan"], d["roofline"]["frac"]),
          "parity", d.get("parity", {}).get("index_equal"), "clk", d["clocks"]["sm_mhz"])
except Exception as e:
    print(t, "failed", e)
PY
done
