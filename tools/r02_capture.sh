#!/bin/bash
# usage (GPU box, repo root): tools/r02_capture.sh
# the round's closing measurements: -m gpu suite, default bench line, the
# reference arm, launch list of one build, --set full of the two scan kernels
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputests.log 2>&1
echo "tests_rc=$?" >> gpurun_out/r02_gputests.log
tail -2 gpurun_out/r02_gputests.log
RNNDG_TRACE=1 timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_trace.err
echo "bench_rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err
echo "ref_rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/r02_launches.csv python tools/prof_build.py > gpurun_out/r02_ncu1.log 2>&1
echo "launches_rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_scan_spec -s 5 -c 1 \
  -o gpurun_out/r02_short_p5 -f python tools/prof_build.py > gpurun_out/r02_ncu2.log 2>&1
echo "short_rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_scan_hub -s 18 -c 1 \
  -o gpurun_out/r02_hub_p18 -f python tools/prof_build.py > gpurun_out/r02_ncu3.log 2>&1
echo "hub_rc=$?"
