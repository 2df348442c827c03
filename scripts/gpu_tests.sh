#!/bin/bash
# GPU test pass: pytest -m gpu (optionally a -k filter / file list), smoke, a short bench.
# usage: scripts/gpu_tests.sh [pytest args...]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/status.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 2400 python -m pytest -m gpu -q --timeout 1200 -p no:cacheprovider -rA "${@:-tests}" \
  > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
tail -3 gpurun_out/pytest_gpu.log
tail -1 gpurun_out/bench.log | cut -c1-600
