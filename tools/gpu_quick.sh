python -m pytest tests -m gpu -x -q > gpurun_out/s2_pytest_gpu.log 2>&1; tail -3 gpurun_out/s2_pytest_gpu.log
for c in c2 c3 c4 c5; do python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value']), 'frac', round(d['roofline']['frac'],3), d['clocks'])"; done
