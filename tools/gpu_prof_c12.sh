CMD="python bench.py --config c12 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-parity --no-sustained --n-elem 256"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2b_launches_c12.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"large_u_xs_kernel" -s 40 -c 1 -o gpurun_out/r2b_c12_u $CMD > gpurun_out/ncu2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"large_(w|v|moments)_kernel" -s 60 -c 3 -o gpurun_out/r2b_c12_wvm $CMD > gpurun_out/ncu3.log 2>&1
echo done $?
