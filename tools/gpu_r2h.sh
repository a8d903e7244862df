python -m pytest tests -m gpu -q > gpurun_out/r2h_pytest_gpu.log 2>&1; tail -4 gpurun_out/r2h_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; tail -2 gpurun_out/r2h_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; tail -2 gpurun_out/r2h_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2h_bench_ref.json 2> gpurun_out/r2h_bench_ref.err
python -c "
import json; d=json.loads(open('gpurun_out/r2h_bench.json').read())
print('c2', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], round(d.get('sustained',{}).get('value',0)), d['e2e']['value'])
for k,v in d.get('configs',{}).items(): print(k, round(v.get('value',0)), v.get('roofline',{}).get('frac'), v.get('parity',{}).get('ok'), v.get('error'))
print(open('gpurun_out/r2h_bench_ref.json').read()[:300])
"
python tools/stage_roofline.py c2 c3 c4 c5 > gpurun_out/r2h_stage_roofline.jsonl 2> /dev/null
python tools/mom_ab.py c5 c12 > gpurun_out/r2h_mom_ab.txt 2>&1; cat gpurun_out/r2h_mom_ab.txt
python tools/grid_perf.py > gpurun_out/r2h_grid_perf.jsonl 2> gpurun_out/r2h_grid_perf.err; tail -2 gpurun_out/r2h_grid_perf.err
B="--no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --no-parity"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 \
    --csv --log-file gpurun_out/r2h_launches_c2.csv python bench.py --steps 2 --warmup 3 $B > gpurun_out/r2h_launches_c2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 \
    --csv --log-file gpurun_out/r2h_launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --n-elem 48 $B > /dev/null 2>&1
