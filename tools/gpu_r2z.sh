# planner sweeps on small / one-CTA fused shapes; the drop-in grid with the new X-chunk policy
P2S_JIT_SWEEP=tools/sweep_small_fused.json python tools/jit_variants.py run > gpurun_out/r2z_sweep_fused.jsonl 2>&1
python - <<EOF
import json
for l in open('gpurun_out/r2z_sweep_fused.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    if 'opts' in d: print(d['case'], d['opts'], d['ok'], round(d['elem_per_s']), round(d['alpha+M GB/s']), d['path'][-90:])
EOF
python tools/grid_perf.py > gpurun_out/r2z_grid_perf.jsonl 2> gpurun_out/r2z_grid_perf.err; tail -2 gpurun_out/r2z_grid_perf.err
python -c "
import json
for l in open('gpurun_out/r2z_grid_perf.jsonl'):
    d=json.loads(l); print(d['shape'], round(d.get('elem_per_s',0)), round(d.get('frac',0),3), d.get('path','')[:40], d.get('error',''))
"
