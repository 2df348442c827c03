#!/bin/bash
# All bench lines (cfg2 with the CPU baseline, cfg3-5, the reference arm)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench_cfg2=$?" >> gpurun_out/status.txt
for wl in cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/bench_$wl.log 2>&1; echo "bench_$wl=$?" >> gpurun_out/status.txt
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "bench_ref=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
