cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/status.txt
nvidia-smi > gpurun_out/nvsmi.txt 2>&1; nproc > gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench_cfg2=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
