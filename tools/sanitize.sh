#!/bin/bash
# compute-sanitizer memcheck / initcheck / synccheck / racecheck over
# tools/sanitize_cases.py, for the default plan choice and forced K12c plans
# (BGS_K12C_PLAN=CR), plus the unmerged / unfused path.  Logs ->
# gpurun_out/sanitize_*.log; one summary line per run.
cd "$(dirname "$0")/.."
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name, tool, env...
  local name=$1 tool=$2; shift 2
  env "$@" timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 99 \
      python tools/sanitize_cases.py ${QUICK:+quick} > gpurun_out/sanitize_${name}.log 2>&1
  echo "$name ($tool $*): rc=$? $(grep -E 'ERROR SUMMARY|failures:' gpurun_out/sanitize_${name}.log | tr '\n' ' ')"
}
run memcheck memcheck BGS_POISON=1
run memcheck_plan21 memcheck BGS_K12C_PLAN=21
run memcheck_plan22 memcheck BGS_K12C_PLAN=22
run memcheck_unmerged memcheck BGS_NO_MERGE_SMALL=1 BGS_NO_FUSE=1
run initcheck initcheck BGS_K12C_PLAN=11
QUICK=1 run synccheck synccheck BGS_K12C_PLAN=14
QUICK=1 run synccheck21 synccheck BGS_K12C_PLAN=21
QUICK=1 run racecheck racecheck BGS_K12C_PLAN=12
QUICK=1 run racecheck21 racecheck BGS_K12C_PLAN=21
