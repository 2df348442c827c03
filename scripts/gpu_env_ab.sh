#!/bin/bash
# A/B of an environment knob on the cfg2 stream bench: scripts/gpu_env_ab.sh VAR=VALUE [bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; : > gpurun_out/env_ab.txt
kv=$1; shift
for rep in 1 2 3; do
  for on in 0 1; do
    if [ $on = 1 ]; then export "$kv"; else unset "${kv%%=*}"; fi
    timeout 600 python bench.py --no-cpu-baseline --no-pce-compare --steps 20 "$@" > gpurun_out/env_run.log 2>&1
    echo "$([ $on = 1 ] && echo "$kv" || echo base) $(tail -1 gpurun_out/env_run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; t=r.get("traffic_measured") or {}; print(round(d["value"]/1e9,2), "e2e", round(d["e2e"]["value"]/1e9,2), " ".join(k+"="+str(round(v,1)) for k,v in r["kernel_ms"].items()), "check MB/frame-iter", round((t.get("bytes_per_frame_iteration") or 0)/1e6,2) if isinstance(t,dict) else t)' 2>&1 | tail -1)" >> gpurun_out/env_ab.txt
  done
done
cat gpurun_out/env_ab.txt
