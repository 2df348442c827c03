#!/bin/bash
# ncu of a mid-stream cfg2 step: plain run first, the launch list of the bench
# command, then one --set full capture (with source) of the five step kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pce-compare --no-traffic > gpurun_out/ncu_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pce-compare --no-traffic > gpurun_out/ncu_launch.log 2>&1
echo "ncu_launches=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_check|k_var|k_decide|k_turnover|k_compact" \
    -s ${SKIP:-60} -c ${COUNT:-5} -o gpurun_out/prof_full python bench.py --traffic-probe --mode stream > gpurun_out/ncu_full.log 2>&1
echo "ncu_full=$?"
