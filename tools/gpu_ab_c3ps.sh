# A/B: C3 two-stage contraction variants (0 default 256 threads; 2-4 parity split with 512 / 512 / 384 threads)
for rep in 1 2; do
for v in 0 2 3 4; do
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --options "P2S_V2_VARIANT=$v" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 v2 variant $v', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], d['roofline']['avg_launch_ms'], d['clocks']['reasons'])"
done; done
