#!/bin/bash
# cfg2 stream: device and e2e edge-updates/s against the number of slots (batches in flight)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out; : > gpurun_out/slots.txt
for rep in 1 2; do
for s in ${SLOTS:-256 384 512 640 768}; do
  timeout 600 python bench.py --no-cpu-baseline --no-pce-compare --no-traffic --steps ${STEPS:-20} --slots $s "$@" > gpurun_out/slots_run.log 2>&1
  echo "slots=$s $(tail -1 gpurun_out/slots_run.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(round(d["value"]/1e9,2), "e2e", round(d["e2e"]["value"]/1e9,2), " ".join(k+"="+str(round(v,1)) for k,v in r["kernel_ms"].items()))' 2>&1 | tail -1)" >> gpurun_out/slots.txt
done
done
cat gpurun_out/slots.txt
