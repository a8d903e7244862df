# CUDA-graph replay of large-path fills: parity test, host-bound check, C5 / c12 bench lines, grid throughput
python -m pytest tests/test_gpu_edges.py -m gpu -q -x -k "graph_replay or concurrent_streams or writes_stay" > gpurun_out/r2ad_pytest.log 2>&1; tail -5 gpurun_out/r2ad_pytest.log
python tools/host_bound.py c12
python tools/host_bound.py c12 0 "P2S_GRAPH=0"
python tools/host_bound.py c5
python tools/host_bound.py c5 0 "P2S_GRAPH=0"
run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --options "$2" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', '$2', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], d['clocks']['reasons'])"; }
run c5 ""; run c12 ""; run c5 "P2S_GRAPH=0"; run c12 "P2S_GRAPH=0"
python tools/grid_perf.py > gpurun_out/r2ad_grid_perf.jsonl 2> gpurun_out/r2ad_grid_perf.err; tail -2 gpurun_out/r2ad_grid_perf.err
python -c "
import json
for l in open('gpurun_out/r2ad_grid_perf.jsonl'):
    d=json.loads(l); print(d['shape'], round(d.get('elem_per_s',0)), round(d.get('frac',0),3), d.get('path','')[:30], d.get('error',''))
"
