# parity of the 43-shape grid after the planner / large-path changes, then its throughput
python -m pytest tests/test_gpu_shapes.py -m gpu -q -x > gpurun_out/r2aa_pytest_shapes.log 2>&1; tail -4 gpurun_out/r2aa_pytest_shapes.log
python tools/grid_perf.py > gpurun_out/r2aa_grid_perf.jsonl 2> gpurun_out/r2aa_grid_perf.err; tail -2 gpurun_out/r2aa_grid_perf.err
python -c "
import json
for l in open('gpurun_out/r2aa_grid_perf.jsonl'):
    d=json.loads(l); print(d['shape'], round(d.get('elem_per_s',0)), round(d.get('frac',0),3), d.get('path','')[:40], d.get('error',''))
"
