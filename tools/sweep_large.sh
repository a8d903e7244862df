#!/bin/bash
# C5 large-path knobs: P2S_LARGE_PS, P2S_LARGE_OVERLAP, P2S_XCHUNK_MB
for ps in 1 0; do for ov in 1 0; do for mb in ${MBS:-32 64}; do
  P2S_LARGE_PS=$ps P2S_LARGE_OVERLAP=$ov P2S_XCHUNK_MB=$mb python bench.py --config c5 --steps ${STEPS:-3} --warmup 3 \
    --no-cpu-baseline --no-e2e --no-ablation 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ps', $ps, 'overlap', $ov, 'xchunk_mb', $mb, round(d['value']), 'frac', round(d['roofline']['frac'],3))"
done; done; done
