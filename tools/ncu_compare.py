"""Side-by-side summary of `ncu --set full --csv --page raw` captures.

usage: python tools/ncu_compare.py label=file.csv [label=file.csv ...]
Prints duration, pipe utilisation (FP64 / DMMA), issue activity, instruction
count, shared wavefronts, DRAM bytes and the top stall reasons per capture.
"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe (DFMA) %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("smsp__inst_executed.sum", "instructions"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("dram__bytes_read.sum", "DRAM read B"),
    ("dram__bytes_write.sum", "DRAM write B"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
]


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    return dict(zip(rows[h], rows[h + 2])), dict(zip(rows[h], rows[h + 1]))


def main(args):
    caps = []
    for a in args:
        label, path = a.split("=", 1)
        caps.append((label, *load(path)))
    w = max(len(l) for l, _, _ in caps)
    print("kernel:", caps[0][1].get("Kernel Name", "")[:100])
    for key, name in KEYS:
        vals = [d.get(key, "n/a") for _, d, _ in caps]
        unit = caps[0][2].get(key, "")
        print(f"  {name:22s}" + "".join(f"  {v:>16s}" for v in vals) + f"  {unit}")
    print("  " + " " * 22 + "".join(f"  {l:>16s}" for l, _, _ in caps))
    for label, d, _ in caps:
        st = {}
        for k, v in d.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
                except ValueError:
                    pass
        top = sorted(st.items(), key=lambda x: -x[1])[:6]
        print(f"  stalls {label:{w}s}: " + " ".join(f"{k}={v:.2f}" for k, v in top))


if __name__ == "__main__":
    main(sys.argv[1:])
