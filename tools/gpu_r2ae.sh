# graph replay + XS u stage for odd N_w + moment k1-chunk heuristic: parity, C5 / c12 bench lines, grid throughput
python -m pytest tests/test_gpu_edges.py tests/test_gpu_shapes.py -m gpu -q -x > gpurun_out/r2ae_pytest.log 2>&1; tail -5 gpurun_out/r2ae_pytest.log
run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --options "$2" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', '$2', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], d['clocks']['reasons'])"; }
run c5 ""; run c12 ""; run c12 "P2S_JIT_KC=4"; run c12 "P2S_JIT_KC=8"
python tools/grid_perf.py > gpurun_out/r2ae_grid_perf.jsonl 2> gpurun_out/r2ae_grid_perf.err; tail -2 gpurun_out/r2ae_grid_perf.err
python -c "
import json
for l in open('gpurun_out/r2ae_grid_perf.jsonl'):
    d=json.loads(l); print(d['shape'], round(d.get('elem_per_s',0)), round(d.get('frac',0),3), d.get('path','')[:30], d.get('error',''))
"
