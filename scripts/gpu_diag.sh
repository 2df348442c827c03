#!/bin/bash
# Diagnostics: tests, probe, bench (clock sampling periods), ncu of the top kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout 600 python scripts/perf_probe.py cfg2 64 > gpurun_out/probe.log 2>&1; echo "probe=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --clock-ms 2000 > gpurun_out/bench_c2000.log 2>&1; echo "bench2=$?" >> gpurun_out/status.txt
python scripts/ncu_target.py cfg2 64 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_check|k_var" -s 4 -c 2 \
    -o gpurun_out/prof_cfg2 python scripts/ncu_target.py cfg2 64 > gpurun_out/ncu_full.log 2>&1
echo "ncu=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
