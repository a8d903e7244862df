"""Print an ncu --metrics CSV launch list as one line per launch."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
out = {}
for r in rows:
    if 'Metric Name' in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    out.setdefault((int(d['ID']), d['Kernel Name'][:50]), {})[d['Metric Name']] = d['Metric Value']
for (i, k), v in sorted(out.items()):
    print(i, k, ' '.join(f"{m.split('__')[1].split('.')[0]}={v[m]}" for m in sorted(v)))
