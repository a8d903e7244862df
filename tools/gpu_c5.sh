# C5 quick check: large-path parity tests, bench at X chunk sizes / u fibers, launch list
python -m pytest tests -m gpu -x -q -k "large or c5 or conforming" 2>&1 | tail -2
for fib in ${FIBS:-2 1}; do for mb in ${MBS:-64 96}; do P2S_LARGE_FIB=$fib P2S_XCHUNK_MB=$mb python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fib $fib xchunk_mb $mb', round(d['value']), round(d['roofline']['frac'],3))"; done; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 10 --csv --log-file gpurun_out/c5_launches.csv python bench.py --config c5 --steps 1 --warmup 3 --n-elem 28 --no-cpu-baseline --no-e2e --no-ablation > /dev/null 2>&1
python tools/launches.py gpurun_out/c5_launches.csv
