#!/bin/bash
# Same-box A/B of one library option (bench.py stage times, 3 rounds
# alternating): tools/ab_opt.sh NAME VALUE_A VALUE_B [CONFIG]
set -u
cd "$(dirname "$0")/.."
N=$1; A=$2; B=$3; C=${4:-cfg5}
for r in 1 2 3; do
  for v in "$A" "$B"; do
    python bench.py --config "$C" --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --dropin-config "" --no-parity \
      --option "$N=$v" > gpurun_out/ab.json 2>/dev/null
    python -c "import json,sys;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$N=$v'.ljust(24), round(d['ms_per_step'],3), d['stage_ms'])"
  done
done
