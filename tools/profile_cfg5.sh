#!/bin/bash
# GPU-box profiling recipe (run under gpurun from the repo root):
#   1. plain bench (must exit 0 before any ncu run)
#   2. launch list (gpu__time_duration per launch, cold/serialised)
#   3. ncu --set full of the hot kernels, one launch each
# Usage: tools/profile_cfg5.sh TAG [KERNEL_REGEX]
set -e
TAG=${1:-cur}
KRE=${2:-"k_tile_segment|k_tt_succ|k_tt_jump|k_tokens_tma|k_brick_tma|k_emit_chunks"}
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
cat gpurun_out/bench_${TAG}.json
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --dropin-config "" --no-parity > gpurun_out/ncu_launch_${TAG}.log 2>&1 || true
ncu --set full --import-source on --clock-control none -k "regex:${KRE}" -c 6 \
    -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --dropin-config "" --no-parity > gpurun_out/ncu_full_${TAG}.log 2>&1 || true
tail -3 gpurun_out/ncu_full_${TAG}.log
