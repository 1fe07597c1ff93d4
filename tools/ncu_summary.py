"""Summarise an ncu --set full capture of the evaluator plus the launch list of a bench run.

  python tools/ncu_summary.py <full.ncu-rep> <launches.csv> <out.json> "<command>" [round]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

rep, launches, out, command = sys.argv[1:5]
rnd = int(sys.argv[5]) if len(sys.argv) > 5 else 2
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
get = lambda name: v[h.index(name)] if name in h else None  # noqa: E731
SCALE = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
         "msecond": 1.0, "second": 1e3, "hz": 1e-9, "khz": 1e-6, "mhz": 1e-3, "ghz": 1.0}


def num(name):
    """Value in base units: bytes, milliseconds, GHz (ncu's raw page carries a unit row)."""
    x = get(name)
    try:
        val = float(str(x).replace(",", ""))
    except (TypeError, ValueError):
        return None
    return val * SCALE.get(units[h.index(name)].strip().lower(), 1.0)


dur_ms = num("gpu__time_duration.sum")
summary = {
    "round": rnd,
    "command": command,
    "kernel": get("Kernel Name") or get("Function Name"),
    "launch": {"grid": num("launch__grid_size"), "block": num("launch__block_size"),
               "registers_per_thread": num("launch__registers_per_thread"),
               "shared_mem_per_block_bytes": num("launch__shared_mem_per_block_dynamic"),
               "occupancy_limit_blocks_per_sm": num("launch__occupancy_limit_shared_mem")},
    "duration_ms": dur_ms,
    "dram_bytes_read": num("dram__bytes_read.sum"),
    "dram_bytes_write": num("dram__bytes_write.sum"),
    "warp_instructions": num("smsp__inst_executed.sum"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "alu_pipe_pct": num("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    "fma_pipe_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "threads_per_warp_instruction": num("smsp__thread_inst_executed_per_inst_executed.ratio"),
    "local_load_instructions": num("smsp__sass_inst_executed_op_local_ld.sum"),
    "shared_load_instructions": num("smsp__sass_inst_executed_op_shared_ld.sum"),
    "sm_clock_ghz": num("smsp__cycles_elapsed.avg.per_second"),
}
stalls = {}
for i, name in enumerate(h):
    if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("_not_issued"):
        try:
            stalls[name[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(v[i].replace(",", ""))
        except ValueError:
            pass
tot_s = sum(stalls.values()) or 1.0
summary["stall_samples_pct"] = {k: round(100 * x / tot_s, 1) for k, x in
                                sorted(stalls.items(), key=lambda kv: -kv[1]) if x / tot_s >= 0.005}
summary["dram_bytes_per_launch"] = (summary["dram_bytes_read"] or 0) + (summary["dram_bytes_write"] or 0)
lrows = [r for r in csv.reader(open(launches)) if len(r) > 10]
lh = lrows[0]
ki, vi = lh.index("Kernel Name"), lh.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in lrows[1:]:
    agg[r[ki]][0] += 1
    agg[r[ki]][1] += float(r[vi].replace(",", "")) / 1e6
tot = sum(x[1] for x in agg.values())
summary["launch_share_in_bench"] = {k: {"launches": n, "total_ms": round(ms, 3), "share": round(ms / tot, 4)}
                                    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])}
json.dump(summary, open(out, "w"), indent=1)
print(json.dumps({k: summary[k] for k in ("kernel", "duration_ms", "issue_active_pct", "warps_active_pct",
                                          "dram_bytes_per_launch", "local_load_instructions")}))
