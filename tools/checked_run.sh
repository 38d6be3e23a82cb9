#!/bin/bash
# The checked build (device bounds checks, paper_2507_21791_b200/_lib_chk) over the small
# parity cases of tools/sanitize_cases.py under every K12c plan and the alternative paths,
# with NaN-poisoned buffers, plus the GPU parity tests that exercise the widest shapes.
# (compute-sanitizer is closed on this pool.)  Summary -> stdout; logs -> gpurun_out/.
cd "$(dirname "$0")/.."
export BGS_LIB_PATH=paper_2507_21791_b200/_lib_chk/libbgs_gpu.so BGS_POISON=1
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 900 python tools/sanitize_cases.py > gpurun_out/checked_${name}.log 2>&1
  echo "$name ($*): rc=$? $(grep -E 'failures:|bgs check' gpurun_out/checked_${name}.log | head -3 | tr '\n' ' ')"
}
run default
for plan in 14 12 11 22 21 41; do run plan$plan BGS_K12C_PLAN=$plan; done
run unfused BGS_NO_FUSE=1
run unmerged BGS_NO_MERGE_SMALL=1
run k2t BGS_K2M=0
run chained BGS_UPDATE_MAXKP=24
run graph0 BGS_GRAPH=0
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "wide or m2048 or factor_matches or plans or chunked or classic or ip1s" > gpurun_out/checked_pytest.log 2>&1
echo "pytest subset under the checked build: rc=$? $(tail -1 gpurun_out/checked_pytest.log)"
