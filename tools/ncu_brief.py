"""Brief per-kernel summary of `ncu --set full --csv --page raw` captures (all kernels in the file)."""
import csv
import sys

KEYS = ['gpu__time_duration.sum', 'launch__registers_per_thread', 'launch__grid_size',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_sectors_srcunit_tex_op_write.sum',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem']
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[h]
    for r in rows[h + 2:]:
        d = dict(zip(hdr, r))
        print(path.split('/')[-1], d['Kernel Name'][:60])
        for k in KEYS:
            print(f"    {k:70s} {d.get(k)}")
        st = []
        for k, v in d.items():
            if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued'):
                try:
                    st.append((float(v.replace(',', '')), k[len('smsp__pcsamp_warps_issue_stalled_'):]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        tot = sum(v for v, _ in st) or 1
        print('    stalls', ', '.join(f"{k} {v / tot:.2f}" for v, k in st[:8]))
