CMD="python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-parity --no-sustained --no-subconfigs --n-elem 64"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"large_u_xs_kernel" -s 6 -c 1 -o gpurun_out/r2_c5_u $CMD > gpurun_out/ncu2.log 2>&1
echo done $?
