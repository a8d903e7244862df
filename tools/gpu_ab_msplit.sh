for cfg in c5 c12; do for ms in 1 0; do
python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --options "P2S_LARGE_MSPLIT=$ms" 2>gpurun_out/ab_err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); E=d['config']['elements_per_rank']; print('$cfg msplit $ms', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], 'moments us/elem', round(1e3*d['stage_ms_per_step']['moments']/E,3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/ab_err.log
done; done
