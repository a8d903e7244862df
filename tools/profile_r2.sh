#!/bin/bash
# Round-2 ncu evidence on one B200 (after the plain runs exited 0): launch list of the default bench
# command, then one --set full capture (source on) of the dominant kernel(s) of C2, C3, C4, C5 and c12.
set -u
R=${ROUND:-r2f}
B="--no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --no-parity"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 \
    --csv --log-file gpurun_out/${R}_launches_c2.csv python bench.py --steps 2 --warmup 3 $B > gpurun_out/${R}_launches_c2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 \
    --csv --log-file gpurun_out/${R}_launches_c3.csv python bench.py --config c3 --steps 1 --warmup 3 --n-elem 8192 $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 \
    --csv --log-file gpurun_out/${R}_launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --n-elem 48 $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 160 \
    --csv --log-file gpurun_out/${R}_launches_c12.csv python bench.py --config c12 --steps 1 --warmup 3 --n-elem 96 $B > /dev/null 2>&1
for c in c2 c4; do
  ncu --set full --import-source on --clock-control none -k regex:fill_fused -s 3 -c 1 -f -o gpurun_out/${R}_ncu_${c}_fused \
      python bench.py --config $c --steps 1 --warmup 3 --n-elem 2048 $B > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:"moments_v2|contract_v2" -s 2 -c 2 -f -o gpurun_out/${R}_ncu_c3_twostage \
    python bench.py --config c3 --steps 1 --warmup 1 --n-elem 4096 $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:large_ -s 4 -c 4 -f -o gpurun_out/${R}_ncu_c5 \
    python bench.py --config c5 --steps 1 --warmup 1 --n-elem 32 $B > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:large_ -s 4 -c 4 -f -o gpurun_out/${R}_ncu_c12 \
    python bench.py --config c12 --steps 1 --warmup 1 --n-elem 96 $B > /dev/null 2>&1
for f in c2_fused c4_fused c3_twostage c5 c12; do
  ncu -i gpurun_out/${R}_ncu_$f.ncu-rep --page raw --csv > gpurun_out/${R}_ncu_${f}_raw.csv 2> /dev/null
  python tools/ncu_summary.py gpurun_out/${R}_ncu_$f.ncu-rep > gpurun_out/${R}_ncu_${f}_summary.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/${R}_ncu_$f.ncu-rep > gpurun_out/${R}_ncu_${f}_sass_hot.txt 2>&1
  rm -f gpurun_out/${R}_ncu_$f.ncu-rep   # 10-50 MB each: gpurun_out/ returns at most 64 MiB
done
python tools/stage_roofline.py c2 c3 c4 c5 > gpurun_out/${R}_stage_roofline.jsonl 2> /dev/null
ls -la gpurun_out/${R}_* | head -40
