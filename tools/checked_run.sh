#!/bin/bash
# The device-bounds-checked build (libplmss_b200_checked.so: every computed
# index into a table, list, bitmap or output of the fused and z-slab passes is
# asserted, fused.cu DCHECK) under the GPU parity suites, full-size configs
# included. Stand-in for compute-sanitizer memcheck, which is closed on the
# GPU pool. Log -> gpurun_out/checked_run.log
#   gpurun --timeout 2400 -- bash tools/checked_run.sh
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export PLMSS_B200_LIB=$PWD/paper_2303_15491_b200/libplmss_b200_checked.so
test -f "$PLMSS_B200_LIB" || { echo "missing $PLMSS_B200_LIB (run __graft_entry__.build())"; exit 2; }
python -c "import paper_2303_15491_b200.api as a; print(\"library:\", a.LIB_PATH)"
timeout 2000 python -m pytest tests/test_full_size.py tests/test_gpu_slab.py tests/test_gpu_parity.py -m gpu -q \
  -k "not streamed" > gpurun_out/checked_run.log 2>&1
echo "checked run rc=$?"
tail -5 gpurun_out/checked_run.log
