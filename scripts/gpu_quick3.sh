#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_quick.sh
timeout 600 python scripts/vnr_pce_sweep.py gpurun_out/vnr_pce_sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep=$?"
bash scripts/gpu_launches.sh
