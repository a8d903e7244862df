# compact Z padding: grid parity + throughput, C5 / c12 sanity, large-path GPU tests
python -m pytest tests/test_gpu_shapes.py -m gpu -q -x > gpurun_out/r2ac_pytest_shapes.log 2>&1; tail -4 gpurun_out/r2ac_pytest_shapes.log
python tools/grid_perf.py > gpurun_out/r2ac_grid_perf.jsonl 2> gpurun_out/r2ac_grid_perf.err; tail -2 gpurun_out/r2ac_grid_perf.err
python -c "
import json
for l in open('gpurun_out/r2ac_grid_perf.jsonl'):
    d=json.loads(l); print(d['shape'], round(d.get('elem_per_s',0)), round(d.get('frac',0),3), d.get('path','')[:30], d.get('error',''))
"
run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --options "$2" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', '$2', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], d['clocks']['reasons'])"; }
run c5 ""; run c12 ""
