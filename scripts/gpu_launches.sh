#!/bin/bash
# per-launch durations of one VNR decode (cfg2, 64 frames) + one PCE D_max=6 decode
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/nt_vnr.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vnr.csv \
    python scripts/ncu_target.py cfg2 64 vnr > gpurun_out/ncu_vnr.log 2>&1
echo "vnr=$?"
