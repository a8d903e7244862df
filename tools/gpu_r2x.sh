# C3: fused 512-thread parity-split variant (7) vs the two-stage default; then the drop-in grid throughput
for rep in 1 2; do
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 default', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], d['kernel_path'][:40])"
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --options "P2S_FUSED_VARIANT=7" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 fused variant 7', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], d['kernel_path'][:40])"
done
python tools/grid_perf.py > gpurun_out/r2x_grid_perf.jsonl 2> gpurun_out/r2x_grid_perf.err; tail -2 gpurun_out/r2x_grid_perf.err
python -c "
import json
for l in open('gpurun_out/r2x_grid_perf.jsonl'):
    d=json.loads(l); print(d['shape'], round(d.get('elem_per_s',0)), round(d.get('frac',0),3), d.get('path','')[:100], d.get('error',''))
"
