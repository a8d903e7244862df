for cfg in c12 c5; do for ub in 1 0; do
python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --options "P2S_LARGE_UBULK=$ub" 2>gpurun_out/ab_err_$cfg$ub.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg ubulk $ub', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], d['parity']['worst_rel_to_block_max'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/ab_err_$cfg$ub.log
done; done
