#!/bin/bash
# tests (non full-size) + perf probe
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout 600 python scripts/perf_probe.py ${1:-cfg2} ${2:-64} > gpurun_out/probe.log 2>&1; echo "probe=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
