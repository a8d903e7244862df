#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   1. default bench line (driver command) + wall time, 2. reference arm,
#   3. ncu launch list of the bench command, 4. ncu --set full (raw CSV) of the
#   dominant kernel per config.  Outputs in gpurun_out/; copy summaries to profiles/.
set -u
mkdir -p gpurun_out
R=${ROUND:-r1}
t0=$(date +%s); python bench.py > gpurun_out/${R}_bench_default.json 2> gpurun_out/${R}_bench_default.err; echo "bench.py default wall: $(( $(date +%s) - t0 )) s" >> gpurun_out/${R}_bench_default.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${R}_bench_reference.json 2> gpurun_out/${R}_bench_reference.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 \
    --csv --log-file gpurun_out/${R}_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    --no-e2e > gpurun_out/${R}_launches_c2.log 2>&1
for c in c2 c4; do
  ncu --set full --clock-control none -k regex:fill_fused -s 3 -c 1 --csv --page raw python bench.py --config $c \
      --steps 1 --warmup 3 --n-elem 2048 --no-cpu-baseline --no-e2e --no-ablation \
      > gpurun_out/${R}_ncu_${c}_fused_raw.csv 2> /dev/null
done
# C3 runs the two-stage path: one moments_v2 and one contract_v2 launch
ncu --set full --clock-control none -k regex:"moments_v2|contract_v2" -s 2 -c 2 --csv --page raw python bench.py \
    --config c3 --steps 1 --warmup 1 --n-elem 4096 --no-cpu-baseline --no-e2e --no-ablation \
    > gpurun_out/${R}_ncu_c3_twostage_raw.csv 2> /dev/null
python tools/stage_roofline.py c1 c2 c3 c4 c5 > gpurun_out/${R}_stage_roofline.jsonl 2> /dev/null
ncu --set full --clock-control none -k regex:large_ -s 4 -c 4 --csv --page raw python bench.py --config c5 \
    --steps 1 --warmup 1 --n-elem 32 --no-cpu-baseline --no-e2e --no-ablation > gpurun_out/${R}_ncu_c5_raw.csv 2> /dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 \
    --csv --log-file gpurun_out/${R}_launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --n-elem 48 \
    --no-cpu-baseline --no-e2e --no-ablation > gpurun_out/${R}_launches_c5.log 2>&1
for c in c3 c4 c5; do python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation \
    > gpurun_out/${R}_bench_$c.json 2> /dev/null; done
ls -la gpurun_out/${R}_*
