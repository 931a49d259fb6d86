#!/bin/bash
# usage (on the GPU box, from the repo root): tools/gpu_check.sh TAG [bench env...]
# runs the -m gpu suite and one traced C3 bench; logs into gpurun_out/
tag=${1:-x}; shift
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_$tag.log 2>&1
echo "tests_rc=$?" >> gpurun_out/gputests_$tag.log
tail -2 gpurun_out/gputests_$tag.log
env RNNDG_TRACE=1 "$@" timeout 300 python bench.py --no-cpu-baseline --no-recall > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{t}.json").readline())
    print("build_s", d["build_seconds"], d["stage_seconds"], "frac", d["roofline"]["frac"])
except Exception as e:
    print("bench failed", e)
PY
