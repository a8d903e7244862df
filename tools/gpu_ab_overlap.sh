for cfg in c12 c5; do for up in -1 2 1; do
python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-parity --options "P2S_LARGE_UPERSIST=$up" 2>gpurun_out/ab_err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg upersist $up', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/ab_err.log
done; done
