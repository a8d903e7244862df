#!/bin/bash
# Fused-kernel variant sweep (P2S_FUSED_VARIANT): usage tools/sweep_fused.sh c2:0,1 c3:0,4
# prints value, roofline frac, SM clock and power per variant
for spec in "$@"; do
  cfg=${spec%%:*}; list=${spec##*:}
  for v in ${list//,/ }; do
    P2S_FUSED_VARIANT=$v python bench.py --config $cfg --steps ${STEPS:-40} --warmup 3 --no-cpu-baseline --no-e2e --no-ablation 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', 'variant', $v, round(d['value']), 'frac', round(d['roofline']['frac'],3), 'sm_mhz', d['clocks'].get('sm_mhz'), 'W', d['clocks'].get('power_w_median'), d['kernel_path'][:60])"
  done
done
