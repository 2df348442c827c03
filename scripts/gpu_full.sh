#!/bin/bash
# Full GPU-box pass: tests, smoke, benches (all workloads + reference arm), launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
rm -f gpurun_out/status.txt
nvidia-smi > gpurun_out/nvsmi.txt 2>&1; nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "bench_cfg2=$?" >> gpurun_out/status.txt
for wl in cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/bench_$wl.log 2>&1; echo "bench_$wl=$?" >> gpurun_out/status.txt
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "bench_ref=$?" >> gpurun_out/status.txt
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pce-compare --no-traffic > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pce-compare --no-traffic > gpurun_out/ncu_launch.log 2>&1
echo "ncu_launches=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
timeout 900 python scripts/vnr_pce_sweep.py gpurun_out/et_sweep_cfg2.json > gpurun_out/sweep2.log 2>&1; echo "sweep2=$?" >> gpurun_out/status.txt
timeout 900 python scripts/vnr_pce_sweep.py gpurun_out/et_sweep_cfg5.json --workload cfg5 > gpurun_out/sweep5.log 2>&1; echo "sweep5=$?" >> gpurun_out/status.txt
python scripts/ncu_target.py cfg2 64 vnr > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_check|k_var|k_decide|k_turnover" -s 8 -c 4 \
    -o gpurun_out/prof_full python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/ncu_full.log 2>&1
echo "ncu_full=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt
