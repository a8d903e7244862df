#!/bin/bash
# Tuning sweep over the registered contraction variants (P2S_V2_VARIANT).
# usage: tools/sweep_variants.sh c2:6 c3:4 c4:3
for spec in "$@"; do
  cfg=${spec%%:*}; n=${spec##*:}
  for ((v=0; v<n; v++)); do
    P2S_V2_VARIANT=$v python bench.py --config $cfg --n-elem 2048 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', 'variant', $v, round(d['value']), 'contract_ms', round(d['stage_ms_per_step']['contract'],3), 'frac', round(d['roofline']['frac'],3), 'mom_ms', round(d['stage_ms_per_step']['moments'],3))" 2>&1 | tail -1
  done
done
