#!/bin/bash
# Round-2 measurement pass on one B200: GPU tests + smoke, every bench line
# (cfg2 stream headline, cfg2 batch, cfg3-5, met, the reference arm, the
# multi-decoder), the guard-build tests, the launch list and one ncu --set
# full capture of the step kernels, the ET sweeps and the QC probe.
# Outputs in gpurun_out/; copy what is judged into profiles/r2/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; : > gpurun_out/status.txt
st() { echo "$1=$2" >> gpurun_out/status.txt; }
nvidia-smi > gpurun_out/nvsmi.txt 2>&1; nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 -p no:cacheprovider -rA -s > gpurun_out/pytest_gpu.log 2>&1; st pytest $?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; st smoke $?
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; st bench_cfg2 $?
timeout 900 python bench.py --mode batch --no-cpu-baseline --no-traffic > gpurun_out/bench_cfg2_batch.log 2>&1; st bench_cfg2_batch $?
for wl in cfg3 cfg4 cfg5 met; do
  timeout 1200 python bench.py --workload $wl --no-cpu-baseline --no-traffic > gpurun_out/bench_$wl.log 2>&1; st bench_$wl $?
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; st bench_ref $?
timeout 900 python bench.py --multi --gpus 1 --workload cfg4 --steps 2 > gpurun_out/bench_multi.log 2>&1; st bench_multi $?
bash scripts/guard_tests.sh > /dev/null 2>&1; st guard $?
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-pce-compare --no-traffic > gpurun_out/ncu_launch.log 2>&1
st ncu_launches $?
ncu --set full --clock-control none --import-source on -k regex:"k_check|k_var|k_decide|k_turnover|k_compact" \
    -s 60 -c 5 -o gpurun_out/prof_full python bench.py --traffic-probe --mode stream > gpurun_out/ncu_full.log 2>&1
st ncu_full $?
timeout 1200 python scripts/vnr_pce_sweep.py gpurun_out/et_sweep_cfg2.json > gpurun_out/sweep2.log 2>&1; st sweep2 $?
timeout 900 python scripts/vnr_pce_sweep.py gpurun_out/et_sweep_cfg5.json --workload cfg5 --no-none > gpurun_out/sweep5.log 2>&1; st sweep5 $?
timeout 900 python scripts/qc_probe.py > gpurun_out/qc.log 2>&1; st qc $?
timeout 1800 python scripts/vnr_pce_sweep.py gpurun_out/et_sweep_met.json --workload met --betas 0.84 0.85 0.86 0.865 0.87 0.875 0.88 0.9 --batches 8 --dmax 250 1000 --no-none > gpurun_out/sweep_met.log 2>&1; st sweep_met $?
timeout 900 python bench.py --multi --gpus 1 --workload cfg5 --frames 8192 --steps 1 --no-traffic > gpurun_out/bench_cfg5_stream8192.log 2>&1; st bench_cfg5_8192 $?
cat gpurun_out/status.txt
