"""Aggregate an ncu source page (cuda,sass) by CUDA source line: stall samples, warp instructions.

  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > /tmp/cs.csv
  python tools/ncu_lines.py /tmp/cs.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
path = None
hdr = None
agg = []
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
        samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        inst = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    stalls = {}
    for k, name in enumerate(hdr):
        if name.startswith("stall_") and "Not Issued" not in name:
            try:
                v = int(r[k])
            except ValueError:
                continue
            if v:
                stalls[name[6:]] = v
    agg.append((samples, inst, f"{path}:{r[0]}", r[1][:70], stalls))
tot_s = sum(a[0] for a in agg) or 1
tot_i = sum(a[1] for a in agg) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, i, loc, src, st in sorted(agg, reverse=True)[:top]:
    main = ", ".join(f"{k}:{v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {loc:18s} {src:70s} [{main}]")
