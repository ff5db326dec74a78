#!/bin/bash
# Same-box comparison of several library variants on one config:
# tools/ab3v.sh CONFIG VARIANT... ("" = the default build)
set -u
cd "$(dirname "$0")/.."
C=$1; shift
for r in 1 2; do
  for V in "$@"; do
    lib=""; [ "$V" != "default" ] && lib="paper_2303_15491_b200/libplmss_b200_${V}.so"
    PLMSS_B200_LIB=$lib python bench.py --config "$C" --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      --dropin-config "" --no-parity > gpurun_out/ab.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$C', '$V'.ljust(8), round(d['ms_per_step'],3), d['stage_ms'])"
  done
done
