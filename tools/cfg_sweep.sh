#!/bin/bash
# tools/cfg_sweep.sh CONFIG "ENV=V ENV2=V2;ENV=V3;..." : one bench line per env set
cfg=$1
IFS=';' read -ra sets <<< "$2"
for st in "${sets[@]}"; do
  env $st timeout 600 python bench.py --config $cfg --steps 2 --warmup 2 --no-cpu-baseline --no-recall > gpurun_out/cs.json 2> gpurun_out/cs.err
  python -c "import json; d=json.loads(open('gpurun_out/cs.json').readline()); print('$cfg [$st]', round(d['build_seconds'],4), round(d['stage_seconds']['scan'],4))" || tail -2 gpurun_out/cs.err
done
