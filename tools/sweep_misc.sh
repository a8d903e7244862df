b() { env "$@" python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$CFG', '$*', round(d['value']), round(d['roofline']['frac'],3))"; }
CFG=c5; b P2S_XCHUNK_MB=96; b P2S_XCHUNK_MB=128; b P2S_XCHUNK_MB=160; b P2S_XCHUNK_MB=96
CFG=c3; b P2S_CHUNK_MB=256; b P2S_CHUNK_MB=512; b P2S_CHUNK_MB=1024; b P2S_CHUNK_MB=256
