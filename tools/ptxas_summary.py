"""Registers / spills per kernel from the ptxas -v log of the build
(build/csrc/p2s_capi.ptxas.log).  Usage: python tools/ptxas_summary.py [filter]"""
import re
import subprocess
import sys

log = open("build/csrc/p2s_capi.ptxas.log").read()
flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
for line in log.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
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
