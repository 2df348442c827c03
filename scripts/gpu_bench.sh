#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for args in "--steps 10" "--steps 3" "--steps 30"; do
  timeout 900 python bench.py --warmup 3 --no-cpu-baseline --no-pce-compare $args > gpurun_out/bench_tmp.log 2>&1
  echo "$args :: $(tail -1 gpurun_out/bench_tmp.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,1), round(d["ms_per_step"],2), round(d["host_ms_per_step"],2), d["warmup_steps_run"], d["clocks"])')"
done
timeout 600 python scripts/perf_probe.py cfg2 64 > gpurun_out/probe.log 2>&1; cut -c1-300 gpurun_out/probe.log
