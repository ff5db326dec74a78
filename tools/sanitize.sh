#!/bin/bash
# compute-sanitizer runs of the fused pipeline and the staged API kernels
# (memcheck / racecheck). Logs -> gpurun_out/sanitize_*.log;
# the summaries worth keeping are copied to profiles/ by hand.
#   gpurun --timeout 1800 -- bash tools/sanitize.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name, tool, args...
  local name=$1 tool=$2
  shift 2
  echo "== $name ($tool)"
  timeout 1500 $CS --tool "$tool" --error-exitcode 9 --print-limit 50 python tools/sanitize_case.py "$@" \
    > "gpurun_out/sanitize_${name}.log" 2>&1
  echo "rc=$?"
  tail -4 "gpurun_out/sanitize_${name}.log"
}
run memcheck_cfg1_spec1 memcheck cfg1 --spec 1 --staged
run memcheck_cfg1_spec0 memcheck cfg1 --spec 0
run memcheck_cfg1_hash memcheck cfg1 --spec 1 --path 2
run memcheck_cfg2_spec0 memcheck cfg2 --spec 0
run racecheck_cfg1 racecheck cfg1 --spec 1
run synccheck_cfg1 synccheck cfg1 --spec 1
run initcheck_cfg1 initcheck cfg1 --spec 1
