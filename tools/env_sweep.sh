#!/bin/bash
# tools/env_sweep.sh VAR "v1 v2 ..." : C3 bench (2 steps) per value of VAR
var=$1
for v in $2; do
  env $var=$v RNNDG_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --no-recall --steps 2 --warmup 3 > gpurun_out/es_${var}_$v.json 2> gpurun_out/es_${var}_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/es_${var}_$v.json').readline()); print('$var=$v', d['build_seconds'], d['stage_seconds']['scan'])" || tail -3 gpurun_out/es_${var}_$v.err
done
