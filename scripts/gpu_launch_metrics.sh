#!/bin/bash
# Per-launch duration, DRAM bytes, instructions and issue activity of the cfg2 VNR decode (ncu, one GPU)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__cycles_active.avg,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launch_metrics.csv python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/ncu_lm.log 2>&1
echo "ncu=$?"
