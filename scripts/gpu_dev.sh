#!/bin/bash
# Development pass on the GPU box: GPU tests (without the full-size ones),
# config-2 perf probe, config-2 and config-3 bench lines, launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_quick.sh
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1; echo "bench_cfg2=$?"
timeout 600 python bench.py --workload cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo "bench_cfg3=$?"
bash scripts/gpu_launches.sh
