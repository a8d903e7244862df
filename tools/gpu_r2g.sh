python -m pytest tests -m gpu -q > gpurun_out/r2g_pytest_gpu.log 2>&1; tail -12 gpurun_out/r2g_pytest_gpu.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; tail -3 gpurun_out/r2g_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2g_bench.json').read())
print('c2', round(d['value']), round(d['roofline']['frac'],3), d['parity'], d.get('sustained',{}).get('value'))
for k,v in d.get('configs',{}).items(): print(k, round(v.get('value',0)), v.get('roofline',{}).get('frac'), v.get('parity',{}).get('ok'), v.get('error'))
print(d['cpu_baseline'])
"
