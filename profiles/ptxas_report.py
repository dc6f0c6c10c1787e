"""Registers / spills per kernel from `nvcc -Xptxas -v` (run here, no GPU)."""
import re
import subprocess
import sys

out = ""
for src in ("engine.cu", "dssync_b200.cu", "problems_abi.cu"):
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-fmad=false",
           "-Xcompiler", "-fPIC", "-Iinclude", "-Ipaper_2007_03298_b200/csrc", "-Xptxas=-v", "-c",
           "paper_2007_03298_b200/csrc/" + src, "-o", "/tmp/ptxas_report.o"]
    out += subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
rows = []
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        spill = m.group(1)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.append((cur, int(m.group(1)), spill))
        cur = None
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for name, regs, spill in rows:
    if pat in name:
        print(f"{regs:4d} regs  spill {spill or 0:>3}B  {name}")
