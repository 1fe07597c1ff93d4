"""Per-kernel registers / spills of one evaluator TU (ptxas -v), demangled template flags.

  python tools/ptxas_report.py [ps_eval_i32_m1.cu]
"""
import os
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(os.environ.get('PTXAS_ROOT') or Path(__file__).resolve().parents[1])
src = ROOT / "paper_2510_05186_b200" / "csrc" / (sys.argv[1] if len(sys.argv) > 1 else "ps_eval_i32_m1.cu")
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O3",
       "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas=-v", "-I", str(ROOT / "include"),
       "-c", str(src), "-o", "/tmp/_ptxas_report.o"]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Function properties for (\S+)", line) or re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows.setdefault(cur, {})["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
names = ["MOVES", "GSTATE", "REC", "DERIVED", "UNI"]
for k, v in rows.items():
    m = re.search(r"eval_kernelI(\w)((?:Lb[01]E){5})", k)
    if m:
        flags = re.findall(r"Lb([01])E", m.group(2))
        tag = " ".join(n for n, f in zip(names, flags) if f == "1") or "-"
        k = f"eval<{m.group(1)}> {tag}"
    print(f"{k[:60]:60s} regs={v.get('regs')} spill(st/ld)={v.get('spill')}")
