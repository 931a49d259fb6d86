#!/bin/bash
# tools/lib_sweep.sh "exp/a.so exp/b.so ..." : C3 bench (2 steps) per library build
for so in $1; do
  t=$(basename $so .so)
  RNNDG_LIB_PATH=$PWD/$so RNNDG_TRACE=1 timeout 300 python bench.py --no-cpu-baseline --no-recall --steps 2 --warmup 3 > gpurun_out/ls_$t.json 2> gpurun_out/ls_$t.err
  python -c "import json; d=json.loads(open('gpurun_out/ls_$t.json').readline()); print('$t', d['build_seconds'], d['stage_seconds']['scan'])" || tail -3 gpurun_out/ls_$t.err
done
