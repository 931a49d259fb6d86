#!/bin/bash
# hub-kernel sweep on the GPU box: tools/hub_sweep.sh "MODE:BIG ..."
for mb in $1; do
  m=${mb%%:*}; b=${mb##*:}
  RNNDG_HUB=$m RNNDG_BIG_HUB=$b RNNDG_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --no-recall --steps 2 --warmup 3 > gpurun_out/sw_$m_$b.json 2> gpurun_out/sw_${m}_$b.err
  python -c "import json; d=json.loads(open('gpurun_out/sw_$m_$b.json').readline()); print('mode $m big $b', d['build_seconds'], d['stage_seconds']['scan'])" || tail -3 gpurun_out/sw_${m}_$b.err
done
