"""Benchmark: candidate schedules evaluated per second (BASELINE.json metric) on config 3.

Workload (BASELINE.json configs[2]): Llama-style 7B
synthetic stage profile, 8 stages x 64 microbatches, PCIe-bandwidth-limited
offload, 65,536 candidates per round per GPU.  A step is one local-search
round: every neighbour of the incumbent is generated on the device, evaluated
by the sm_100a evaluator kernel, reduced to the best (makespan, index) key,
all-reduced (MIN) across ranks, and the winner applied on improvement.
Scaling is weak: each rank owns 65,536 neighbours of every round.

Keys beyond the driver contract:
  roofline      INT32-issue roofline of the evaluator kernel: algorithmic
                work 10 int ops per committed event over the kernel's CUDA-event time, against
                the INT32 peak measured live by ps_int32_probe on the same GPU.
  cpu_baseline  the C restatement of the reference algorithm (oracle/, "port"), all host
                threads, on the first neighbours of the same round; parity of that sample
                with the GPU is checked and reported.
  e2e           the same metric through the C ABI with HOST buffers: the round's neighbours as
                differences from the incumbent (ps_eval_batch_host_delta) in pinned host memory,
                copied in, rebuilt and evaluated with the incumbent as base, results copied out,
                every step; e2e_rows the same with full stage rows (ps_eval_batch_host), and
                e2e_no_base full rows with no base (every candidate simulated in full).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate schedules evaluated/sec"
UNIT = "candidates/s"
CONFIG = 3
PER_GPU = 65536
SEED = 20251005
MOVES = dict(shift_permille=700, max_shift=4)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class ClockSampler:
    """SM clock and throttle reasons sampled during the timed region: NVML every 5 ms (the timed
    region is a fraction of a second), nvidia-smi every 200 ms when NVML is unavailable."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[index]) if vis and vis.split(",")[index].isdigit() else index
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(phys))
        except Exception:
            self._nvml = None

    def _run_nvml(self):
        nv, h = self._nvml
        masks = [nv.nvmlClocksThrottleReasonHwSlowdown, nv.nvmlClocksThrottleReasonHwThermalSlowdown,
                 nv.nvmlClocksThrottleReasonSwThermalSlowdown, nv.nvmlClocksThrottleReasonSwPowerCap]
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append([str(self.index), str(sm), str(mx)] +
                                 ["Active" if r & mk else "Not Active" for mk in masks])
            except Exception:
                pass
            self._stop.wait(0.005)

    def _run(self):
        if self._nvml is not None:
            return self._run_nvml()
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def build_incumbent_oracle(inst, pk, orc):
    """AdaOffload structure found with the CPU port (first feasible fill of the back-off sequence)."""
    import numpy as np
    from paper_2510_05186_b200.heuristics import ada_backoff_sequence, filled_order
    from paper_2510_05186_b200.packing import encode_candidate
    off = frozenset(inst.offloadable_ops())
    for fills in ada_backoff_sequence(inst):
        o, mk, _ = encode_candidate(pk, {i: filled_order(inst, i, fills[i]) for i in range(1, pk.num_stages + 1)}, off)
        r = orc.run(o, mk)
        if r["flags"] == 1:
            return o, mk, r["makespan"]
    raise RuntimeError("no feasible AdaOffload structure")


def calibrate_sample(orc, inc_o, inc_m, rnd, threads, target_s, cap):
    """Neighbour count whose CPU evaluation takes about target_s seconds on `threads` threads
    (timed on a sample of 8 candidates per thread: per-candidate costs vary several-fold)."""
    k = min(cap, 8 * threads)
    t = time.perf_counter()
    orc.search_round(inc_o, inc_m, SEED, MOVES["shift_permille"], MOVES["max_shift"], rnd, 0, k, threads)
    per = (time.perf_counter() - t) / k                   # wall seconds per candidate, all threads
    n = int(target_s / max(per, 1e-7))
    return max(threads, min(cap, n))


def _philox_np(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 over numpy arrays (the move decode of DESIGN.md §4, host-side analysis only)."""
    import numpy as np
    M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    c0, c1, c2, c3 = [np.asarray(x, np.uint32) for x in (c0, c1, c2, c3)]
    for r in range(10):
        if r:
            k0 = (k0 + 0x9E3779B9) & 0xFFFFFFFF
            k1 = (k1 + 0xBB67AE85) & 0xFFFFFFFF
        p0 = M0 * c0.astype(np.uint64)
        p1 = M1 * c2.astype(np.uint64)
        c0, c1, c2, c3 = ((p1 >> np.uint64(32)).astype(np.uint32) ^ c1 ^ np.uint32(k0), p1.astype(np.uint32),
                          (p0 >> np.uint64(32)).astype(np.uint32) ^ c3 ^ np.uint32(k1), p0.astype(np.uint32))
    return c0, c1, c2, c3


def distinct_move_fraction(inst, rounds, neighbours):
    """Share of a round's neighbours that are distinct moves (adjacent shifts a<->a+1 coincide;
    no-ops coincide), averaged over `rounds` — what a deduplicating CPU search would simulate."""
    import numpy as np
    from paper_2510_05186_b200 import OpId, OpKind
    P, m, L = inst.num_stages, inst.num_microbatches, 3 * inst.num_microbatches
    offl = np.array([[inst.act_size.get(OpId(s + 1, j + 1, OpKind.F), 0) > 0 for j in range(m)]
                     for s in range(P)])
    any_off = bool(offl.any())
    idx = np.arange(neighbours, dtype=np.uint64)
    fr = []
    for rnd in rounds:
        r0, r1, r2, r3 = _philox_np(idx.astype(np.uint32), (idx >> np.uint64(32)).astype(np.uint32),
                                    np.full(neighbours, rnd & 0xFFFFFFFF, np.uint32),
                                    np.full(neighbours, rnd >> 32, np.uint32), SEED & 0xFFFFFFFF, SEED >> 32)
        st = (r1 % P).astype(np.int64)
        shift = (~np.bool_(any_off)) | ((r0 % 1000) < MOVES["shift_permille"])
        a = (r2 % L).astype(np.int64)
        d = 1 + ((r3 >> 1) % MOVES["max_shift"]).astype(np.int64)
        b = np.clip(np.where(r3 & 1, a - d, a + d), 0, L - 1)
        j = (r2 % m).astype(np.int64)
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        adj = (hi - lo) == 1
        key = np.where(shift, np.where(b == a, -1, (st * 8192 + np.where(adj, lo, a)) * 8192 + np.where(adj, hi, b)),
                       np.where(offl[st, j], -2 - (st * m + j), -1))
        fr.append(len(np.unique(key)) / neighbours)
    return float(np.mean(fr))


def run_reference(args):
    """--impl reference: the reference algorithm's CPU restatement (oracle port), all host threads."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Oracle
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.packing import pack_instance
    inst = workloads.CONFIGS[CONFIG]()
    pk = pack_instance(inst)
    orc = Oracle(pk)
    threads = cpu_threads()
    inc_o, inc_m, _ = build_incumbent_oracle(inst, pk, orc)
    # each step a bounded sample: the whole --steps/--warmup run stays within ~2.5 minutes
    step_s = min(args.ref_step_seconds, 150.0 / max(1, args.steps + args.warmup))
    cap = PER_GPU * max(1, args.gpus)
    n = calibrate_sample(orc, inc_o, inc_m, 0, threads, step_s, cap)
    for w in range(args.warmup):
        t = time.perf_counter()
        orc.search_round(inc_o, inc_m, SEED, MOVES["shift_permille"], MOVES["max_shift"], w, 0, n, threads)
        # re-size the sample from the measured warm-up throughput
        n = max(threads, min(cap, int(step_s * n / max(time.perf_counter() - t, 1e-3))))
    times = []
    for k in range(args.steps):
        t = time.perf_counter()
        orc.search_round(inc_o, inc_m, SEED, MOVES["shift_permille"], MOVES["max_shift"],
                         args.warmup + k, 0, n, threads)
        times.append(time.perf_counter() - t)
    total = sum(times)
    value = n * args.steps / total
    sample = f"first {n} neighbours of each round (of {PER_GPU * max(1, args.gpus)}), config {CONFIG} warm-start incumbent"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": workload_config(args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(world):
    from paper_2510_05186_b200 import workloads
    inst = workloads.CONFIGS[CONFIG]()
    doc = " ".join((workloads.CONFIGS[CONFIG].__doc__ or "").split())
    return {"workload": f"config{CONFIG}: {doc} AdaOffload/best_feasible incumbent, {PER_GPU} neighbours/round/GPU",
            "stages": inst.num_stages, "microbatches": inst.num_microbatches, "candidates_per_round": PER_GPU * world,
            "candidates_per_gpu": PER_GPU, "parallelism": f"candidates sharded over {world} GPU(s)",
            "l2": "flushed (256 MiB write) between timed steps",
            "moves": MOVES, "seed": SEED}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-seconds", type=float, default=3.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ttb", action="store_true")
    ap.add_argument("--ttb-rounds", type=int, default=1000)
    ap.add_argument("--ils-seconds", type=float, default=10.0)
    # other BASELINE configs for manual runs (the driver's line is config 3, 65,536 per GPU)
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--per-gpu", type=int, default=65536)
    args = ap.parse_args()
    global CONFIG, PER_GPU
    CONFIG, PER_GPU = args.config, args.per_gpu
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2510_05186_b200 import _native as N, workloads
    from paper_2510_05186_b200.heuristics import best_feasible
    from paper_2510_05186_b200.listsched import stage_order_of
    from paper_2510_05186_b200.search import LocalSearch, SearchConfig

    rank, world, local = dist_env()
    # PS_SHARE_GPU=1 (tests only): several ranks on one device over gloo, to exercise the sharded
    # path where only one GPU is available; the product path is one rank per GPU over NCCL
    share = os.environ.get("PS_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    inst = workloads.CONFIGS[CONFIG]()
    s0, gen_name = best_feasible(inst, device=local)
    orders0 = {i: stage_order_of(s0, i) for i in range(1, inst.num_stages + 1)}
    cfg = SearchConfig(seed=SEED, neighbours=PER_GPU * world, **MOVES)
    ls = LocalSearch(inst, orders0, s0.offloaded, cfg, device=local)
    lib, di = ls.lib, ls.di
    events_total = torch.zeros(2, dtype=torch.int64, device=dev)   # [simulated, algorithmic] events
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def round_timed(ev_k0, ev_k1):
        ls.best_key.fill_(N.BEST_NONE)
        desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), ls.round, ls.first,
                            ls.count, ls.moves, events_total.data_ptr(),
                            ls.base.handle if ls.base is not None else None)
        ev_k0.record(stream)
        if ls.nccl_comm:
            # over NCCL the 8-byte all-reduce(MIN) runs inside the C ABI call, after the kernels
            N.check(lib.ps_search_round_sharded(di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()), None,
                                                C.c_void_p(ls.nccl_comm), C.c_void_p(stream.cuda_stream)))
            ev_k1.record(stream)
        else:
            N.check(lib.ps_search_round(di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()), None,
                                        C.c_void_p(stream.cuda_stream)))
            ev_k1.record(stream)
            if world > 1:
                dist.all_reduce(ls.best_key, op=dist.ReduceOp.MIN)
        return ls.finish_round()

    # ---- warm-up -------------------------------------------------------------------------------
    for _ in range(args.warmup):
        round_timed(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed search rounds -----------------------------------------------------------------------
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    improved = 0
    events_total.zero_()
    with ClockSampler(local) as clk:
        for k in range(K):
            flush.fill_(k & 0xFF)          # evict L2 between steps (outside the step events)
            es0, ek0, ek1, es1 = evs[k]
            es0.record(stream)
            improved += bool(round_timed(ek0, ek1))
            es1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [evs[k][0].elapsed_time(evs[k][3]) for k in range(K)]
    kern_ms = [evs[k][1].elapsed_time(evs[k][2]) for k in range(K)]
    print(json.dumps({"diag_step_ms": [round(x, 2) for x in step_ms], "diag_kern_ms": [round(x, 2) for x in kern_ms]}),
          file=sys.stderr, flush=True)
    total_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    total_s = float(total_ms.item()) / 1e3
    value = cfg.neighbours * K / total_s
    # per round: the divergence-order kernel and its radix sort (CUB, compiled into our library:
    # histogram, exclusive sum, one onesweep pass per 8 key bits — the keys need the bits of 3Pm),
    # the evaluator's main pass and its two overflow passes; per improvement: apply_move, the base
    # re-recording and its checkpoint shift (profiles/r02_launches.csv)
    span = inst.num_stages * 3 * inst.num_microbatches
    key_bits = 1
    while key_bits < 32 and span >> key_bits:
        key_bits += 1
    per_round = 1 + 2 + (key_bits + 7) // 8 + 3
    launches = per_round * K + 3 * improved

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": 1000 * total_s / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": workload_config(world), "clocks": clk.summary(), "gpu_launches": launches}

    # ---- roofline: INT32 issue ----------------------------------------------------
    ev_sim, ev_full = (int(x) for x in events_total.tolist())
    kern_s = sum(kern_ms) / 1e3 / K
    # W_c = 10 int ops per event of every evaluated candidate, E_c = 3Pm + 2|off_c|
    ops_per_launch = 10 * ev_full / K
    probe = torch.zeros(1, dtype=torch.int64, device=dev)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    N.check(lib.ps_int32_probe(200, C.c_void_p(probe.data_ptr()), C.c_void_p(stream.cuda_stream)))
    probe.zero_()
    p0.record(stream)
    N.check(lib.ps_int32_probe(4000, C.c_void_p(probe.data_ptr()), C.c_void_p(stream.cuda_stream)))
    p1.record(stream)
    torch.cuda.synchronize()
    int32_peak = int(probe.item()) / (p0.elapsed_time(p1) / 1e3) / 1e12
    achieved = ops_per_launch / kern_s / 1e12
    # dram__bytes_read.sum + dram__bytes_write.sum of this kernel from the committed ncu --set full
    # capture of the same command (ncu cannot run inside the timed bench)
    traffic, traffic_src, hw = None, None, None
    prof_name = {3: "ncu_eval_summary.json", 5: "ncu_eval_config5_summary.json"}.get(
        CONFIG, "ncu_eval_config%d_summary.json" % CONFIG)
    prof = os.path.join(ROOT, "profiles", prof_name)
    if os.path.exists(prof):
        try:
            doc = json.load(open(prof))
            traffic = doc.get("dram_bytes_per_launch")
            traffic_src = f"profiles/{prof_name} (round {doc.get('round')}, {doc.get('kernel')})"
            # what the hardware was doing in that capture: the kernel is issue-bound, not idle
            hw = {k: doc.get(k) for k in ("issue_active_pct", "alu_pipe_pct", "warps_active_pct",
                                          "threads_per_warp_instruction", "warp_instructions", "duration_ms")}
            hw["source"] = traffic_src
        except Exception:
            traffic = None
    n_cand = cfg.neighbours // world
    hbm_peak, hbm_src = 7700.0, "B200_PROFILING.md nominal (MEASURED_PEAKS.json absent)"
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        hbm_src = "MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth)"
    except Exception:
        pass
    line["roofline"] = {
        "bound": "int32-issue", "achieved": achieved, "peak": int32_peak, "unit": "Tops/s",
        "frac": achieved / int32_peak, "traffic": traffic, "traffic_source": traffic_src,
        "kernel": "ps::eval_kernel<int, moves, smem state, derived channels, symmetric tables> (search round)",
        "kernel_ms_per_launch": 1000 * kern_s, "kernel_share_of_step": sum(kern_ms) / sum(step_ms),
        "ncu_utilisation": hw,
        "algorithmic_events_per_launch": ev_full / K, "simulated_events_per_launch": ev_sim / K,
        "int_ops_per_event": 10,
        "peak_source": "ps_int32_probe measured live on this GPU (IADD3/LOP3/IMAD chains)",
        "hbm": {"algorithmic_bytes_per_launch": n_cand * (16 + 20 + 8 * inst.num_stages),
                "achieved_gbs": n_cand * (16 + 20 + 8 * inst.num_stages) / kern_s / 1e9,
                "peak_gbs": hbm_peak, "peak_gbs_source": hbm_src,
                "note": "not the binding roof: move-encoded candidates"},
        "note": "latency-bound discrete-event simulation (SURVEY.md 8(d)): achieved counts the algorithmic "
                "work of every evaluated candidate (10 int ops x its 3Pm + 2|off| events for a feasible one; a "
                "deadlocked one only with the events committed before the deadlock was concluded, a lower "
                "bound of what the reference commits before it raises); prefix and suffix sharing simulate "
                "only simulated_events_per_launch of them"}

    # ---- e2e through the C ABI with host buffers --------------------------------------------------
    if not args.no_e2e:
        pk = di.packed
        orders_d, masks_d = ls.materialize(ls.first, n_cand)
        torch.cuda.synchronize()
        # uint8 op codes when they fit (4m <= 256): the candidates cross PCIe in half the bytes
        u8 = 4 * pk.num_microbatches <= 256
        h_orders = torch.empty(orders_d.shape, dtype=torch.uint8 if u8 else torch.int16, pin_memory=True)
        h_masks = torch.empty(masks_d.shape, dtype=torch.int32, pin_memory=True)
        h_orders.copy_(orders_d.to(torch.uint8) if u8 else orders_d)
        h_masks.copy_(masks_d)
        outs = dict(makespan=torch.empty(n_cand, dtype=torch.int64, pin_memory=True),
                    bubble=torch.empty(n_cand, dtype=torch.float64, pin_memory=True),
                    flags=torch.empty(n_cand, dtype=torch.int32, pin_memory=True),
                    peak=torch.empty((n_cand, pk.num_stages), dtype=torch.int64, pin_memory=True))
        # the search's outputs (makespan, bubble, STRICT peaks, flags) — no OrderInfeasible stage
        # sets, which no caller of a batch needs and which let deadlocks be concluded early
        cb = N.CandBatch(n_cand, h_orders.data_ptr(), h_masks.data_ptr(), None, 0,
                         ls.base.handle if ls.base is not None else None, 1 if u8 else 2)
        rb = N.ResultBatch(outs["makespan"].data_ptr(), outs["bubble"].data_ptr(), outs["peak"].data_ptr(),
                           outs["flags"].data_ptr(), None, None, None, 0, None)
        h2d = h_orders.numel() * h_orders.element_size() + h_masks.numel() * 4
        d2h = n_cand * (8 + 8 + 4 + 8 * pk.num_stages)
        for _ in range(args.warmup):
            N.check(lib.ps_eval_batch_host(di.handle, C.byref(cb), C.byref(rb), C.c_void_p(stream.cuda_stream)))
        if world > 1:
            dist.barrier()
        e_ms = []
        for k in range(K):
            flush.fill_(k & 0xFF)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            N.check(lib.ps_eval_batch_host(di.handle, C.byref(cb), C.byref(rb), C.c_void_p(stream.cuda_stream)))
            e_ms.append(1000 * (time.perf_counter() - t0))
        e_tot = torch.tensor([sum(e_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e_tot, op=dist.ReduceOp.MAX)
        e_s = float(e_tot.item()) / 1e3
        line["e2e_rows"] = {"value": n_cand * world * K / e_s, "unit": UNIT, "h2d_bytes_per_step": h2d,
                            "d2h_bytes_per_step": d2h, "ms_per_step": 1000 * e_s / K,
                            "api": "ps_eval_batch_host (full stage rows, uint8 codes when m <= 64; pinned host "
                                   "buffers, copies inside the call)",
                            "outputs": "makespan, bubble, per-stage STRICT peak, flags per candidate"}
        e2e_flags = outs["flags"].numpy().copy()
        e2e_span = outs["makespan"].numpy().copy()
        # the headline e2e: the same neighbours in the compact host form, differences from the
        # incumbent (ps_delta_batch: only those cross PCIe; rebuilt in HBM by a kernel)
        from paper_2510_05186_b200.packing import delta_encode
        ref_o = ls.inc_orders.cpu().numpy().view(np.uint16).copy()
        ref_m = ls.inc_mask.cpu().numpy().view(np.uint32).copy()
        enc = delta_encode(ref_o, ref_m, orders_d.cpu().numpy().view(np.uint16), masks_d.cpu().numpy().view(np.uint32))
        pinned = []
        for a in (ref_o, ref_m) + tuple(enc):
            t = torch.empty(a.nbytes, dtype=torch.uint8, pin_memory=True)
            t.numpy()[:] = np.ascontiguousarray(a).view(np.uint8).ravel()
            pinned.append(t)
        db = N.DeltaBatch(n_cand, *[t.data_ptr() for t in pinned], ls.base.handle if ls.base is not None else None)
        h2d_d = sum(t.numel() for t in pinned)
        for _ in range(args.warmup):
            N.check(lib.ps_eval_batch_host_delta(di.handle, C.byref(db), C.byref(rb), C.c_void_p(stream.cuda_stream)))
        if world > 1:
            dist.barrier()
        d_ms = []
        for k in range(K):
            flush.fill_(k & 0xFF)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            N.check(lib.ps_eval_batch_host_delta(di.handle, C.byref(db), C.byref(rb), C.c_void_p(stream.cuda_stream)))
            d_ms.append(1000 * (time.perf_counter() - t0))
        d_tot = torch.tensor([sum(d_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(d_tot, op=dist.ReduceOp.MAX)
        d_s = float(d_tot.item()) / 1e3
        same_d = bool((outs["makespan"].numpy() == e2e_span).all() and (outs["flags"].numpy() == e2e_flags).all())
        line["e2e"] = {"value": n_cand * world * K / d_s, "unit": UNIT, "h2d_bytes_per_step": h2d_d,
                       "d2h_bytes_per_step": d2h, "ms_per_step": 1000 * d_s / K,
                       "api": "ps_eval_batch_host_delta: pinned host buffers holding the neighbours as differences "
                              "from the incumbent (ps_delta_batch), copied in, classified on the device (a candidate "
                              "that is one move of the incumbent runs on the move-encoded kernel against its "
                              "recorded base, any other is rebuilt and evaluated materialised), results copied out, "
                              "every step",
                       "outputs": "makespan, bubble, per-stage STRICT peak, flags per candidate",
                       "outputs_equal_to_e2e_rows": same_d}
        # the same batch as a generic one: no recorded base, every candidate simulated from its
        # first event, like the CPU port (the like-for-like ratio against cpu_baseline)
        cb0 = N.CandBatch(n_cand, h_orders.data_ptr(), h_masks.data_ptr(), None, 0, None, 1 if u8 else 2)
        N.check(lib.ps_eval_batch_host(di.handle, C.byref(cb0), C.byref(rb), C.c_void_p(stream.cuda_stream)))
        k0 = max(1, min(K, 5))
        n_ms = []
        for k in range(k0):
            flush.fill_(k & 0xFF)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            N.check(lib.ps_eval_batch_host(di.handle, C.byref(cb0), C.byref(rb), C.c_void_p(stream.cuda_stream)))
            n_ms.append(1000 * (time.perf_counter() - t0))
        n_tot = torch.tensor([sum(n_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(n_tot, op=dist.ReduceOp.MAX)
        same = bool((outs["makespan"].numpy() == e2e_span).all() and (outs["flags"].numpy() == e2e_flags).all())
        line["e2e_no_base"] = {"value": n_cand * world * k0 / (float(n_tot.item()) / 1e3), "unit": UNIT,
                               "steps": k0, "ms_per_step": float(n_tot.item()) / k0,
                               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                               "outputs_equal_to_e2e": same,
                               "note": "ps_eval_batch_host on full rows without a recorded base: no prefix/suffix "
                                       "sharing, each candidate simulated in full (like the CPU port); e2e and "
                                       "e2e_rows resume from the incumbent's checkpoints"}
    else:
        line["e2e"] = None

    # ---- CPU baseline (rank 0, N=1): the oracle port on the first neighbours of one round ---------------
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle.oracle import Oracle
        pk = di.packed
        orc = Oracle(pk)
        threads = cpu_threads()
        inc_o = ls.inc_orders.cpu().numpy().view(np.uint16)
        inc_m = ls.inc_mask.cpu().numpy().view(np.uint32)
        rnd = ls.round
        n = calibrate_sample(orc, inc_o, inc_m, rnd, threads, args.cpu_seconds, n_cand)
        t0 = time.perf_counter()
        best_cpu, ms_cpu = orc.search_round(inc_o, inc_m, SEED, MOVES["shift_permille"], MOVES["max_shift"],
                                            rnd, 0, n, threads, want_makespans=True)
        cpu_s = time.perf_counter() - t0
        # parity of the sample: the GPU's makespans for the same neighbours of the same round
        ms_gpu = torch.empty(n_cand, dtype=torch.int64, device=dev)
        ls.best_key.fill_(N.BEST_NONE)
        desc = N.SearchDesc(ls.inc_orders.data_ptr(), ls.inc_mask.data_ptr(), rnd, 0, n_cand, ls.moves, None,
                            ls.base.handle if ls.base is not None else None)
        N.check(lib.ps_search_round(di.handle, C.byref(desc), C.c_void_p(ls.best_key.data_ptr()),
                                    C.c_void_p(ms_gpu.data_ptr()), C.c_void_p(stream.cuda_stream)))
        torch.cuda.synchronize()
        gpu_ms = ms_gpu.cpu().numpy()
        mism = int((gpu_ms[:n] != ms_cpu).sum())
        line["cpu_baseline"] = {"value": n / cpu_s, "unit": UNIT, "cores": threads, "kind": "port",
                                "cpu_model": cpu_model(),
                                "sample": f"first {n} of {n_cand} neighbours of round {rnd} "
                                          f"(C restatement of listsched.run_order, oracle/ps_oracle.c)",
                                "parity": {"checked": n, "makespan_mismatches": mism,
                                           "best_key_equal_on_sample": bool(
                                               int(ms_cpu[ms_cpu >= 0].min() if (ms_cpu >= 0).any() else -1) ==
                                               int(gpu_ms[:n][gpu_ms[:n] >= 0].min() if (gpu_ms[:n] >= 0).any() else -1))}}
        if not args.no_e2e:
            line["e2e"]["feasible_share"] = float((e2e_flags & 1).mean())
    # ---- time to best (BASELINE metric, second half): a fresh search from the same warm start,
    # rounds until 16 in a row bring nothing (or the round cap), wall clock per strict improvement --
    if not args.no_ttb:
        ls2 = LocalSearch(inst, orders0, s0.offloaded, cfg, device=local)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        stale = 0
        r_ms = []
        while ls2.round < args.ttb_rounds and stale < 16:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ls2.launch_round()
            e1.record(stream)
            stale = 0 if ls2.finish_round(t0) else stale + 1
            r_ms.append(e0.elapsed_time(e1))
        elapsed = time.perf_counter() - t0
        last = ls2.improvements[-1] if ls2.improvements else None
        ttb = {"initial_makespan": ls2.initial_makespan, "best_makespan": ls2.makespan,
               "improvement_pct": 100.0 * (ls2.initial_makespan - ls2.makespan) / ls2.initial_makespan,
               "rounds": ls2.round, "improvements": len(ls2.improvements),
               "rounds_to_best": (last.round + 1) if last else 0,
               "seconds_to_best": last.timestamp if last else 0.0, "search_seconds": elapsed,
               "stopped_by": "16 rounds without improvement" if stale >= 16 else f"round cap {args.ttb_rounds}",
               "neighbours_per_round": cfg.neighbours,
               "ms_per_round_mean": sum(r_ms) / len(r_ms), "ms_per_round_last50": sum(r_ms[-50:]) / len(r_ms[-50:]),
               "note": "LocalSearch as shipped: a move drawn several times in a round is simulated once "
                       "(lowest index; DESIGN.md 3.7); the trajectory is that of evaluating every neighbour"}
        if "cpu_baseline" in line:
            ttb["cpu_port_seconds_to_best_estimate"] = ttb["rounds_to_best"] * cfg.neighbours / line["cpu_baseline"]["value"]
            # the same search on the CPU with the same deduplication of repeated moves
            frac = distinct_move_fraction(inst, range(4), cfg.neighbours)
            ttb["distinct_move_fraction"] = frac
            ttb["cpu_port_seconds_to_best_estimate_dedup"] = ttb["cpu_port_seconds_to_best_estimate"] * frac
        line["time_to_best"] = ttb
        # the iterated local search past the descent's convergence, same warm start
        cfg_ils = SearchConfig(seed=SEED, neighbours=PER_GPU * world, kick_moves=4, **MOVES)
        ls4 = LocalSearch(inst, orders0, s0.offloaded, cfg_ils, device=local)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        res4 = ls4.run(time_budget=args.ils_seconds)
        marks = [t for t in (0.5, 1.0, 2.0, 5.0, 10.0, 30.0) if t <= args.ils_seconds]
        at = {str(t): min([ls4.initial_makespan] + [i.makespan for i in res4.improvements if i.timestamp <= t])
              for t in marks}
        line["time_to_best_ils"] = {"seconds": args.ils_seconds, "best_makespan": res4.makespan,
                                    "best_at_seconds": at, "rounds": ls4.round, "kicks": ls4.kicks,
                                    "kick_moves": 4, "improvement_pct": 100.0 * (ls4.initial_makespan - res4.makespan)
                                    / ls4.initial_makespan,
                                    "note": "descent + kicks from the best (DESIGN.md 4.1) for a fixed wall-clock "
                                            "budget; the descent alone stops at its local optimum (time_to_best)"}
    # ---- whole search without deduplication: every neighbour of every round simulated, rounds from
    # the warm start to convergence (the early rounds of `value` are the cheapest ones) ------------
    if not args.no_ttb:
        cfg_nd = SearchConfig(seed=SEED, neighbours=PER_GPU * world, dedup=False, prune=False, **MOVES)
        ls3 = LocalSearch(inst, orders0, s0.offloaded, cfg_nd, device=local)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        round_ms, stale = [], 0
        while ls3.round < args.ttb_rounds and stale < 16:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ls3.launch_round()
            e1.record(stream)
            stale = 0 if ls3.finish_round() else stale + 1      # (host sync: e1 has completed)
            round_ms.append(e0.elapsed_time(e1))
        tot = torch.tensor([sum(round_ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        tail = round_ms[-50:]
        line["value_whole_search"] = {
            "value": cfg_nd.neighbours * len(round_ms) / (float(tot.item()) / 1e3), "unit": UNIT,
            "rounds": len(round_ms), "final_makespan": ls3.makespan, "initial_makespan": ls3.initial_makespan,
            "ms_per_round_mean": float(tot.item()) / len(round_ms),
            "ms_per_round_last50": sum(tail) / len(tail),
            "value_last50": cfg_nd.neighbours * len(tail) / (sum(tail) / 1e3),
            "note": "fresh search from the warm start to 16 rounds without improvement, no move "
                    "deduplication (every neighbour simulated), device time of each round's "
                    "generate + evaluate + argmin (+ all-reduce)"}
    # ---- the Python drop-in per call (encode, one launch, decode into a Schedule) -----------------
    if rank == 0 and not args.no_ttb:
        from paper_2510_05186_b200.heuristics import best_feasible as bf
        from paper_2510_05186_b200.listsched import run_order
        run_order(inst, orders0, s0.offloaded, device=local)
        t0 = time.perf_counter()
        reps = 10
        for _ in range(reps):
            run_order(inst, orders0, s0.offloaded, device=local)
        ro_ms = 1000 * (time.perf_counter() - t0) / reps
        t0 = time.perf_counter()
        bf(inst, device=local)
        bf_ms = 1000 * (time.perf_counter() - t0)
        line["drop_in"] = {"run_order_ms_per_call": ro_ms, "best_feasible_ms_per_call": bf_ms,
                           "note": "listsched.run_order / heuristics.best_feasible as a Python caller sees "
                                   "them: structure encode, one kernel launch, trace decode into a Schedule"}
    line["search"] = {"initial_makespan": ls.initial_makespan, "final_makespan": ls.makespan,
                      "warm_start": gen_name, "rounds": ls.round,
                      "improvements": [[imp.round, imp.makespan] for imp in ls.improvements]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
