#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_turnover" -c 1 \
    -o gpurun_out/prof_turn python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/ncu_turn.log 2>&1
echo "turn=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_compact" -s ${1:-21} -c 1 \
    -o gpurun_out/prof_compact python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/ncu_compact.log 2>&1
echo "compact=$?"
