#!/bin/bash
# GPU tests against the guard build (make guard -> libbpdec_guard.so): every
# device allocation poisoned (0xFF: NaN / -1) and fenced by 64 KiB guard
# zones that are verified at the end of every C-ABI call (csrc/devmem.hpp).
# Out-of-bounds writes fail the call; out-of-bounds or uninitialised reads
# surface as NaN / -1 in outputs that the parity tests compare with the CPU
# reference.  (compute-sanitizer is not available on this GPU pool.)
# usage (GPU box): scripts/guard_tests.sh [pytest args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
export BPDEC_LIB="$PWD/paper_2507_03509_b200/libbpdec_guard.so"
test -f "$BPDEC_LIB" || { echo "missing $BPDEC_LIB (make guard)"; exit 2; }
args=("$@")
[ ${#args[@]} -eq 0 ] && args=(tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_fuzz.py tests/test_harness.py)
timeout 2400 python -m pytest -m gpu -q -p no:cacheprovider -rA "${args[@]}" \
  > gpurun_out/guard_tests.log 2>&1
rc=$?
echo "guard tests rc=$rc"
tail -3 gpurun_out/guard_tests.log
exit $rc
