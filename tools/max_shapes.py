"""The ABI's size limits (PS_MAX_STAGES = 32, PS_MAX_MICROBATCHES = 4096) end to end: generator
structures evaluated on the GPU against the oracle, then search rounds with a recorded base
(every neighbour's makespan against the oracle's).

  python tools/max_shapes.py [P m n_neighbours rounds]...   (default: a fixed list; JSON lines)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.oracle import Oracle  # noqa: E402
from paper_2510_05186_b200 import make_uniform_instance  # noqa: E402
from paper_2510_05186_b200.engine import DeviceInstance  # noqa: E402
from paper_2510_05186_b200.heuristics import generator_structures  # noqa: E402
from paper_2510_05186_b200.packing import delta_encode, encode_candidate, pack_instance  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402


def run(P, m, n, rounds):
    t0 = time.time()
    inst = make_uniform_instance(P, m, 3, 2, 2, 1, 4, 2, 6)
    pk = pack_instance(inst)
    di = DeviceInstance(inst, packed=pk)
    structs = generator_structures(inst)
    enc = [encode_candidate(pk, o, f) for o, f in structs]
    orders = np.stack([e[0] for e in enc])
    masks = np.stack([e[1] for e in enc])
    res = di.evaluate(torch.from_numpy(orders.view(np.int16)).cuda(), torch.from_numpy(masks.view(np.int32)).cuda(),
                      peak=True)
    torch.cuda.synchronize()
    t_gpu = time.time() - t0
    orc = Oracle(pk)
    # the oracle replays only the structure the search starts from (the C port needs minutes for
    # some generator structures at these sizes: its ledger scans are linear)
    flags = res.flags.cpu().numpy().astype(np.uint32)
    ok = flags == 1
    k = int(np.flatnonzero(ok)[-1]) if ok.any() else len(structs) - 1
    t1 = time.time()
    want = orc.eval_batch(orders[k:k + 1], masks[k:k + 1])
    t_orc = time.time() - t1
    eq = bool(flags[k] == want["flags"][0] and int(res.makespan[k].item()) == int(want["makespan"][0]) and
              (not ok[k] or (res.peak[k].cpu().numpy() == want["peak"][0]).all()))
    out = {"P": P, "m": m, "structures": len(structs), "feasible": int(ok.sum()), "eval_equal": eq,
           "eval_seconds": round(t_gpu, 2), "oracle_eval_seconds": round(t_orc, 2)}
    if ok.any() and n > 0:
        o, f = structs[k]
        t1 = time.time()
        ls = LocalSearch(inst, o, f, SearchConfig(seed=5, neighbours=n, shift_permille=700, max_shift=4))
        torch.cuda.synchronize()
        out["search_setup_seconds"] = round(time.time() - t1, 2)
        t_gpu_rounds = t_cpu_rounds = 0.0
        ms = torch.empty(n, dtype=torch.int64, device="cuda")
        checked, bad, bad_delta = 0, 0, 0
        for _ in range(rounds):
            inc_o = ls.inc_orders.cpu().numpy().view(np.uint16).copy()
            inc_m = ls.inc_mask.cpu().numpy().view(np.uint32).copy()
            t1 = time.time()
            ls.launch_round(ms)
            torch.cuda.synchronize()
            t_gpu_rounds += time.time() - t1
            t1 = time.time()
            best, want_ms = orc.search_round(inc_o, inc_m, 5, 700, 4, ls.round, 0, n, want_makespans=True)
            t_cpu_rounds += time.time() - t1
            bad += int((ms.cpu().numpy() != want_ms).sum())
            # the same neighbours as a delta-encoded host batch (moves or rebuilt rows)
            mo, mm = ls.materialize(0, n, ls.round)
            d = delta_encode(inc_o, inc_m, mo.cpu().numpy().view(np.uint16), mm.cpu().numpy().view(np.uint32))
            r = ls.di.evaluate_host_delta(inc_o, inc_m, *d, peak=False, base=ls.base)
            bad_delta += int((np.asarray(r.makespan) != want_ms).sum())
            checked += n
            assert int(ls.best_key.item()) == best
            t1 = time.time()
            ls.finish_round()
            torch.cuda.synchronize()
            out["finish_seconds"] = round(out.get("finish_seconds", 0) + time.time() - t1, 2)
        out.update({"gpu_round_seconds": round(t_gpu_rounds, 2), "oracle_round_seconds": round(t_cpu_rounds, 2),"search_checked": checked, "search_mismatches": bad, "delta_mismatches": bad_delta, "final_makespan": ls.makespan,
                    "initial_makespan": ls.initial_makespan})
    out["seconds"] = round(time.time() - t0, 1)
    return out


if __name__ == "__main__":
    args = [int(a) for a in sys.argv[1:]]
    shapes = [tuple(args[i:i + 4]) for i in range(0, len(args), 4)] or \
        [(32, 1024, 64, 2), (32, 2048, 16, 1), (8, 4096, 32, 2), (1, 4096, 256, 3), (32, 4096, 0, 0)]
    for s in shapes:
        try:
            print(json.dumps(run(*s)), flush=True)
        except Exception as e:  # report and continue with the next shape
            print(json.dumps({"P": s[0], "m": s[1], "error": f"{type(e).__name__}: {e}"[:300]}), flush=True)
