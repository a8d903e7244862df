python -m pytest tests -m gpu -q > gpurun_out/r2f_pytest_gpu.log 2>&1; tail -4 gpurun_out/r2f_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; tail -2 gpurun_out/r2f_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; tail -2 gpurun_out/r2f_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2f_bench_ref.json 2> gpurun_out/r2f_bench_ref.err
python -c "
import json; d=json.loads(open('gpurun_out/r2f_bench.json').read())
print('c2', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], round(d.get('sustained',{}).get('value',0)), d['e2e']['value'])
for k,v in d.get('configs',{}).items(): print(k, round(v.get('value',0)), v.get('roofline',{}).get('frac'), v.get('parity',{}).get('ok'), v.get('error'))
print(open('gpurun_out/r2f_bench_ref.json').read()[:300])
"
