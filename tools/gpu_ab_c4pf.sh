# A/B: C4 default (variant 0) vs the same kernel with the L2 prefetch of the next unit's alpha (variant 7)
for rep in 1 2 3; do
for v in 0 7; do
python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --options "P2S_FUSED_VARIANT=$v" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 variant $v', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], d['clocks']['reasons'])"
done; done
