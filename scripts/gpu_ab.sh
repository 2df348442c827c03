#!/bin/bash
# A/B of an env knob on the cfg2 bench (device value only): run as  gpu_ab.sh VAR=VALUE
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/ab.txt
for rep in 1 2 3; do
  for mode in base alt; do
    if [ $mode = alt ]; then export $1; else unset ${1%%=*}; fi
    timeout 600 python bench.py --no-cpu-baseline --no-pce-compare ${BENCH_ARGS} > gpurun_out/ab_$mode.log 2>&1
    echo "$mode $(tail -1 gpurun_out/ab_$mode.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,2), round(d["ms_per_step"],3), round(d["e2e"]["value"]/1e9,2))')" >> gpurun_out/ab.txt
  done
done
cat gpurun_out/ab.txt
