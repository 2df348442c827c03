#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
timeout 1500 python -m pytest tests/test_harness.py tests/test_gpu_parity.py -m gpu -q --timeout 900 -p no:cacheprovider -x -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout 600 python scripts/perf_probe.py cfg2 64 > gpurun_out/probe.log 2>&1; echo "probe=$?" >> gpurun_out/status.txt
python scripts/ncu_target.py cfg2 64 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_syndrome|k_terminate|k_check|k_var" -s 8 -c 4 \
    -o gpurun_out/prof2_cfg2 python scripts/ncu_target.py cfg2 64 > gpurun_out/ncu_full.log 2>&1
echo "ncu=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
