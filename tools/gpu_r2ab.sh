# v-step n1 slicing (P2S_LARGE_VSPLIT waves; 0 = off) on C5 / c12, the 10x1x14 launch list, grid parity + throughput
run() { python bench.py --config $1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-ablation --no-sustained --no-subconfigs --options "$2" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', '$2', round(d['value']), round(d['roofline']['frac'],3), d['parity']['ok'], d['clocks']['reasons'])"; }
for v in 0 2 4 8; do run c5 "P2S_LARGE_VSPLIT=$v"; run c12 "P2S_LARGE_VSPLIT=$v"; done
python -m pytest tests/test_gpu_shapes.py -m gpu -q -x > gpurun_out/r2ab_pytest_shapes.log 2>&1; tail -4 gpurun_out/r2ab_pytest_shapes.log
python tools/grid_perf.py > gpurun_out/r2ab_grid_perf.jsonl 2> gpurun_out/r2ab_grid_perf.err; tail -2 gpurun_out/r2ab_grid_perf.err
python -c "
import json
for l in open('gpurun_out/r2ab_grid_perf.jsonl'):
    d=json.loads(l); print(d['shape'], round(d.get('elem_per_s',0)), round(d.get('frac',0),3), d.get('path','')[:30], d.get('error',''))
"
# SYMB / IG parity (small shapes + C3 variants), C3 A/B of the two-CTA variants, launch lists of the slowest grid shapes
for i in 37 19 29; do
python tools/grid_one.py $i
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 240 --csv --log-file gpurun_out/r2y_launches_$i.csv python tools/grid_one.py $i 0 1 > /dev/null 2>&1
python - <<EOF
import csv,io,collections
txt=open('gpurun_out/r2y_launches_$i.csv').read().splitlines()
k=[j for j,l in enumerate(txt) if l.startswith('"ID"')][0]
rows=list(csv.DictReader(io.StringIO('\n'.join(txt[k:]))))
agg=collections.OrderedDict()
for r in rows:
    key=(r['ID'], r['Kernel Name'][:60]); agg.setdefault(key,{})[r['Metric Name']]=r['Metric Value']
seen=collections.OrderedDict()
for (id_,name),m in agg.items():
    d=seen.setdefault(name,{'n':0,'t':0.0,'grid':m.get('launch__grid_size'),'blk':m.get('launch__block_size'),'regs':m.get('launch__registers_per_thread')})
    d['n']+=1; d['t']+=float(m.get('gpu__time_duration.sum','0').replace(',',''))
for name,d in seen.items(): print('   ',name, d)
EOF
done
