#!/bin/bash
# Same-box A/B of two builds of the library (bench.py stage times, 3 rounds
# alternating): tools/ab.sh VARIANT [CONFIG] [extra bench args]
#   VARIANT: paper_2303_15491_b200/libplmss_b200_VARIANT.so (_build.build_cuda(variant=..., defines=...))
set -u
cd "$(dirname "$0")/.."
V=$1; C=${2:-cfg5}; shift; shift || true
for r in 1 2 3; do
  for lib in "" "paper_2303_15491_b200/libplmss_b200_${V}.so"; do
    PLMSS_B200_LIB=$lib python bench.py --config "$C" --steps 10 --warmup 3 --no-e2e --no-cpu-baseline \
      --dropin-config "" --no-parity "$@" > gpurun_out/ab.json 2>/dev/null
    python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('${lib:-default}'.ljust(48), round(d['ms_per_step'],3), d['stage_ms'])"
  done
done
