"""Registers and spills per kernel instance from `nvcc -Xptxas -v` output.
Usage: python scripts/ptxas_report.py <source.cu> [name-substring]"""
import re
import subprocess
import sys

src = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else ""
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
       "-std=c++17", "--expt-relaxed-constexpr", "-Xptxas", "-v", "-c", src, "-o", "/dev/null"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr.splitlines()
name = None
spill = None
for line in out:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        spill = None
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and name:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and name:
        if pat in name:
            print(f"{int(m.group(1)):4d} regs  spill st/ld {spill}  {name[:110]}")
        name = None
