# large-path X chunk x u-stage CTAs/SM sweep (c12), C5 reference point
for up in -1 2; do for mb in 96 40 32 24; do
python bench.py --config c12 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-parity --no-sustained --options "P2S_XCHUNK_MB=$mb;P2S_LARGE_UPERSIST=$up" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c12 upersist $up xchunk $mb', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
for mb in 96 128; do
python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-parity --no-sustained --options "P2S_XCHUNK_MB=$mb" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 xchunk $mb', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
