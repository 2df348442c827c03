#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
timeout 600 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench_cfg2=$?"
