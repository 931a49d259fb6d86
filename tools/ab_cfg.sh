#!/bin/bash
# usage (GPU box, repo root): tools/ab_cfg.sh CONFIG TAG "ENV=.." [TAG2 "ENV.."]...
# one bench (2 timed builds) of CONFIG per variant; summary line per variant
cfg=$1; shift
while [ $# -ge 2 ]; do
  tag=$1; envs=$2; shift 2
  env $envs RNNDG_TRACE=1 timeout 600 python bench.py --config $cfg --no-cpu-baseline --no-recall --steps 2 --warmup 1 > gpurun_out/abc_$tag.json 2> gpurun_out/abc_$tag.err
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/abc_{t}.json").readline())
    print(t, "build_s %.4f scan %.4f frac %.4f" % (d["build_seconds"], d["stage_seconds"]["scan"], d["roofline"]["frac"]),
          "parity", (d.get("parity") or {}).get("index_equal"), "checks", d["pair_checks_per_build"])
except Exception as e:
    print(t, "failed", e)
PY
done
