"""Registers / spills per kernel from the ptxas -v logs of the build
(build/csrc/*.ptxas.log).  Usage: python tools/ptxas_summary.py [filter]"""
import glob
import re
import subprocess
import sys

log = "\n".join(open(f).read() for f in sorted(glob.glob("build/csrc/*.ptxas.log")))
flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(anonymous namespace\)::", "", cur)
        cur = re.sub(r"\(int\)|p2s::|\(.*\)$", "", cur)
        continue
    if cur and "spill stores" in line:
        sp = re.search(r"(\d+) bytes spill stores", line).group(1)
        spill = sp
    m = re.search(r"Used (\d+) registers", line)
    if cur and m:
        if flt in cur:
            print(f"{m.group(1):>4} regs  spill {spill:>5} B  {cur[:150]}")
        cur = None
