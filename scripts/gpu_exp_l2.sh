cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/plain.log 2>&1
for f in 0 32 64 128; do
BPDEC_L2_FETCH=$f ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:"k_" --csv --log-file gpurun_out/lm_$f.csv python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/ncu_lm_$f.log 2>&1
done
