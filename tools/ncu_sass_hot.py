"""Hot SASS instructions / stall totals from `ncu -i rep --page source --csv --print-source sass`."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[h]
recs = [dict(zip(hdr, r)) for r in rows[h + 1:] if len(r) == len(hdr) and r[0] != "Address"]
tot = sum(int(r["Warp Stall Sampling (All Samples)"]) for r in recs) or 1
stall_cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(int(r[c]) for r in recs) for c in stall_cols}
print("total samples", tot)
print("stalls:", ", ".join(f"{c[6:]} {v / tot:.2f}" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
op = {}
for r in recs:
    o = r["Source"].split()[0] if r["Source"].split() else "?"
    if o.startswith("@"):
        o = r["Source"].split()[1]
    o = o.split(".")[0]
    op[o] = op.get(o, 0) + int(r["Warp Stall Sampling (All Samples)"])
print("samples by opcode:", ", ".join(f"{k} {v / tot:.2f}" for k, v in sorted(op.items(), key=lambda x: -x[1])[:12]))
ex = {}
for r in recs:
    toks = r["Source"].split()
    o = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
    try:
        ex[o] = ex.get(o, 0) + int(r["Instructions Executed"].replace(",", ""))
    except ValueError:
        pass
etot = sum(ex.values()) or 1
print("executed warp-instructions", etot)
print("executed by opcode:", ", ".join(f"{k} {v / etot:.3f}" for k, v in sorted(ex.items(), key=lambda x: -x[1])[:16]))
recs.sort(key=lambda r: -int(r["Warp Stall Sampling (All Samples)"]))
for r in recs[:top]:
    s = int(r["Warp Stall Sampling (All Samples)"])
    top_st = sorted(((int(r[c]), c[6:]) for c in stall_cols), reverse=True)[:2]
    print(f"{s / tot:6.3f} {r['Address'][-5:]} {r['Source'].strip()[:60]:60s} {top_st}")
