#!/bin/bash
# GPU-box check: parity tests, smoke, perf probe, short bench.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/status.txt
timeout 600 python scripts/perf_probe.py cfg2 64 > gpurun_out/probe.log 2>&1; echo "probe=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --steps 3 --warmup 2 ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
