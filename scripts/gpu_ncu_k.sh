#!/bin/bash
# ncu --set full of kernels matching $1 in the cfg2 VNR decode (skip $2, count $3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/ncu_target.py cfg2 64 vnr > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${2:-10} -c ${3:-1} \
    -o gpurun_out/prof_k python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/ncu_k.log 2>&1
echo "ncu=$?"
