#!/bin/bash
# Development A/B: perf_probe with each exp_libs/lib_*.so in turn.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cp paper_2507_03509_b200/libbpdec.so /tmp/libbpdec_orig.so
for f in exp_libs/lib_*.so; do
  cp $f paper_2507_03509_b200/libbpdec.so
  echo "== $f" >> gpurun_out/exp.log
  timeout 300 python scripts/perf_probe.py ${1:-cfg2} ${2:-64} 2>&1 | cut -c1-420 >> gpurun_out/exp.log
done
cp /tmp/libbpdec_orig.so paper_2507_03509_b200/libbpdec.so
