#!/bin/bash
# A/B of library builds: each exp_libs/*.so in turn (BPDEC_LIB), interleaved,
# REPS rounds, on the bench workload (device value + per-kernel CUDA-event ms).
# usage (GPU box): scripts/gpu_ab_libs.sh [bench args]   env: REPS (default 3)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; : > gpurun_out/ab_libs.txt
for rep in $(seq 1 ${REPS:-3}); do
  for lib in exp_libs/*.so; do
    BPDEC_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-pce-compare --no-traffic --steps 20 "$@" \
      > gpurun_out/ab_run.log 2>&1
    echo "$(basename $lib) $(tail -1 gpurun_out/ab_run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]/1e9,2), round(d["ms_per_step"],3), " ".join(k+"="+str(round(v,1)) for k,v in r["kernel_ms"].items()))' 2>&1 | tail -1)" >> gpurun_out/ab_libs.txt
  done
done
cat gpurun_out/ab_libs.txt
