#!/bin/bash
# A/B of library builds on the QC probe (scripts/qc_probe.py): each exp_libs/*.so in turn
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; : > gpurun_out/ab_qc.txt
for rep in $(seq 1 ${REPS:-2}); do
  for lib in exp_libs/*.so; do
    BPDEC_LIB=$PWD/$lib timeout 900 python scripts/qc_probe.py > gpurun_out/ab_qc_run.log 2>&1
    echo "$(basename $lib) $(python -c 'import json; d=json.load(open("gpurun_out/qc_probe.json")); print({k: {m: round(v["edge_updates_per_s"]/1e9,1) for m,v in d[k].items() if isinstance(v, dict)} for k in d})')" >> gpurun_out/ab_qc.txt
  done
done
cat gpurun_out/ab_qc.txt
