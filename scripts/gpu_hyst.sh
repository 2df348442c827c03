#!/bin/bash
# cfg2 stream against the compaction hysteresis (BPDEC_COMPACT_HYST)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; : > gpurun_out/hyst.txt
for rep in 1 2; do
for h in ${HYST:-2 4 8 12 16 24}; do
  BPDEC_COMPACT_HYST=$h timeout 600 python bench.py --no-cpu-baseline --no-pce-compare --no-traffic --steps 20 "$@" > gpurun_out/hyst_run.log 2>&1
  echo "hyst=$h $(tail -1 gpurun_out/hyst_run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]/1e9,2), "e2e", round(d["e2e"]["value"]/1e9,2), " ".join(k+"="+str(round(v,1)) for k,v in r["kernel_ms"].items()))' 2>&1 | tail -1)" >> gpurun_out/hyst.txt
done
done
cat gpurun_out/hyst.txt
