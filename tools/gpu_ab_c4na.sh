# A/B: C4 default (variant 0) vs the same kernel with alpha loads that do not allocate in L1 (variant 2)
for rep in 1 2; do
for v in 0 2; do
python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --options "P2S_FUSED_VARIANT=$v" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 variant $v', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], d['kernel_path'][-60:])"
done; done
for v in 0 2; do
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_miss.sum,l1tex__t_sectors_pipe_lsu_mem_local_op_ld_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control none -k regex:fill_fused -c 2 --csv --log-file gpurun_out/c4na_v$v.csv python bench.py --config c4 --n-elem 2048 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --no-parity --options "P2S_FUSED_VARIANT=$v" > /dev/null 2>&1
grep -v "^==" gpurun_out/c4na_v$v.csv | awk -F, 'NR>1{print $(NF-2), $(NF)}' | tr -d '"' | tail -6
done
