python -m pytest tests/test_gpu_shapes.py tests/test_gpu_edges.py -m gpu -q -x > gpurun_out/r2g_pytest.log 2>&1; tail -3 gpurun_out/r2g_pytest.log
python tools/grid_perf.py > gpurun_out/r2g_grid_perf.jsonl 2> gpurun_out/r2g_grid_perf.err; tail -2 gpurun_out/r2g_grid_perf.err
python -c "
import json
for l in open('gpurun_out/r2g_grid_perf.jsonl'):
    d=json.loads(l); print(d['shape'], round(d.get('elem_per_s',0)), round(d.get('frac',0),3), d.get('path','')[:30], d.get('error',''))
"
