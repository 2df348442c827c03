#!/bin/bash
# streaming check: cfg4 code, 4096 frames through 512 / 1024 slots; cfg5 8192-frame stream through 1024 slots
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --workload cfg4 --frames 4096 --steps 3 --warmup 3 --no-cpu-baseline --no-pce-compare > gpurun_out/bench_cfg4_4096.log 2>&1; echo "cfg4_4096=$?"
timeout 900 python bench.py --workload cfg5 --frames 8192 --slots 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-pce-compare > gpurun_out/bench_cfg5_8192.log 2>&1; echo "cfg5_8192=$?"
