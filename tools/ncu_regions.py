"""Aggregate an ncu source page (cuda,sass) of eval_kernel by kernel region (line ranges of
ps_eval.cuh found from marker comments/lambdas): warp instructions and stall samples.

  python tools/ncu_regions.py /tmp/cs.csv
"""
import csv
import re
import sys
from collections import defaultdict
from pathlib import Path

SRC = Path(__file__).resolve().parent.parent / "paper_2510_05186_b200/csrc/ps_eval.cuh"
lines = SRC.read_text().splitlines()
marks = [("prologue", r"^template <typename V, bool MOVES, int GS"),
         ("fetch/row helpers", r"auto row_at = "), ("window fold/insert", r"auto win_fold = "),
         ("window tau", r"auto win_tau = "), ("compute_key", r"auto compute_key = "),
         ("transfer_key", r"auto transfer_key = "), ("put_result", r"auto put_result = "),
         ("checkpoint regs", r"auto save_regs = "), ("convergence compare", r"auto diff_dead = "),
         ("work loop", r"const long long n_items = "), ("init: zero/stage/validate", r"=+ initialise"),
         ("init: divergence+restore", r"prefix sharing: the first step"),
         ("init: pruning setup", r"Bound pruning \(search rounds"),
         ("event loop", r"=+ simulate: one committed"), ("finish", r"=+ finished or deadlocked")]
starts = []
for name, rx in marks:
    for k, l in enumerate(lines, 1):
        if re.search(rx, l):
            starts.append((k, name))
            break
starts.sort()


def region(n):
    r = "headers"
    for k, name in starts:
        if n >= k:
            r = name
    return r


rows = list(csv.reader(open(sys.argv[1])))
path, hdr = None, None
ins, smp = defaultdict(int), defaultdict(int)
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r or not r[0] or r[0] == "Function Name":
        continue
    try:
        s = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        i = int(r[hdr.index("Instructions Executed")])
        n = int(r[0])
    except (ValueError, IndexError):
        continue
    key = region(n) if path == "ps_eval.cuh" else f"({path})"
    ins[key] += i
    smp[key] += s
ti, ts = sum(ins.values()) or 1, sum(smp.values()) or 1
print(f"total warp instructions {ti:.4g}, samples {ts}")
for k in sorted(ins, key=lambda x: -ins[x]):
    print(f"{k:28s} {100*ins[k]/ti:5.1f}% ins  {100*smp[k]/ts:5.1f}% smp")
