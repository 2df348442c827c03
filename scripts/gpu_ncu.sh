#!/bin/bash
# ncu capture of the top kernels (one GPU): plain run first, then ncu.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
WL=${WL:-cfg2}
python scripts/ncu_target.py $WL 64 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_check|k_var" -s 4 -c 2 \
    -o gpurun_out/prof_${WL} python scripts/ncu_target.py $WL 64 > gpurun_out/ncu_full.log 2>&1
echo "ncu=$?"
python scripts/ncu_target.py $WL 64 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${WL}.csv python scripts/ncu_target.py $WL 64 > gpurun_out/ncu_launches.log 2>&1
echo "ncu_launches=$?"
