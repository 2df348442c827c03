#!/bin/bash
# A/B of exp_libs/*.so in stream and batch mode (and another workload): scripts/gpu_ab_modes.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; : > gpurun_out/ab_modes.txt
for rep in $(seq 1 ${REPS:-2}); do
  for args in "--mode stream" "--mode batch" "--workload met --steps 8"; do
    for lib in exp_libs/*.so; do
      BPDEC_LIB=$PWD/$lib timeout 600 python bench.py --no-cpu-baseline --no-pce-compare --no-traffic --steps 20 $args \
        > gpurun_out/ab_run.log 2>&1
      echo "$(basename $lib) [$args] $(tail -1 gpurun_out/ab_run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]/1e9,2), round(d["ms_per_step"],3), " ".join(k+"="+str(round(v,1)) for k,v in r["kernel_ms"].items()), d["clocks"]["reasons"])' 2>&1 | tail -1)" >> gpurun_out/ab_modes.txt
    done
  done
done
cat gpurun_out/ab_modes.txt
