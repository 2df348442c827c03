#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_quick.sh
timeout 600 python scripts/perf_probe.py cfg3 32 > gpurun_out/probe_cfg3.log 2>&1; echo "probe3=$?"
timeout 600 python bench.py --workload cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo "bench_cfg3=$?"
