#!/bin/bash
# GPU pass used while iterating: the GPU tests, smoke, then the cfg2 bench (no CPU leg)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/status.txt
timeout 900 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_cfg2.log 2>&1; echo "bench_cfg2=$?" >> gpurun_out/status.txt
tail -1 gpurun_out/bench_cfg2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("BENCH", d["value"]/1e9, d["e2e"]["value"]/1e9, d["roofline"]["frac"], {k: round(v,1) for k,v in d["roofline"]["kernel_ms"].items()}, d["d_bar_vnr"], d["clocks"]["sm_mhz"])' >> gpurun_out/status.txt
cat gpurun_out/status.txt
