# large path sweeps: X chunk size (c12) and CTA slots of the persistent u grid left free for the w / v steps
run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --no-parity --options "$2" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', '$2', round(d['value']), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for x in 8 12 16 20 24; do run c12 "P2S_XCHUNK_MB=$x"; done
for r in 0 12 24 48 74; do run c12 "P2S_LARGE_URESERVE=$r"; done
for r in 0 8 16 32 48; do run c5 "P2S_LARGE_URESERVE=$r"; done
for r in 0 16 32; do run c5 "P2S_LARGE_URESERVE=$r;P2S_XCHUNK_MB=48"; done
for r in 0 16 32; do run c5 "P2S_LARGE_URESERVE=$r;P2S_LARGE_PRIO=1"; done
run c4 ""
