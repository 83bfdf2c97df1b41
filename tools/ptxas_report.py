"""Registers / spills per kernel: python tools/ptxas_report.py <file.cu> [name-filter]"""
import re
import subprocess
import sys

src = sys.argv[1]
filt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++20", "-Xcompiler", "-fPIC",
                      "--expt-relaxed-constexpr", "-Xptxas", "-v", "-c", src, "-o", "/dev/null"],
                     capture_output=True, text=True, cwd=sys.argv[3] if len(sys.argv) > 3 else None).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        rows[cur]["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows[cur]["regs"] = int(m.group(1))
for k, v in rows.items():
    short = re.sub(r"_ZN3akb\d+_GLOBAL__N__\w+?_cu_\w+?\d+", "", k)[:70]
    if filt in k:
        print(f"{short:72s} regs={v.get('regs')} spill={v.get('spill', 0)}")
