"""Reference answers at the BASELINE benchmark shapes (configs 3, 4, 5).

Run here (the reference is importable only in the build container):

    python tests/golden/make_bench_golden.py [3] [4] [5]

For each config it fixes an incumbent structure and a search round, decodes
neighbours of that round with the search's move definition (the
C restatement in oracle/ is used only to decode moves, never to answer), and
runs every neighbour through the UNMODIFIED reference ``pipesched.run_order``
+ ``makespan`` + ``memory_trace(STRICT)`` + the cli.py:156 bubble.  Recorded
per neighbour: (round, index), the move as a diff against the incumbent, the
makespan, the bubble ``repr``, the peaks, ``OrderInfeasible.stages`` and a
SHA-256 of the commit-ordered event trace (the full trace for the first few).

* config 3 (8 x 64 Llama-7B): the bench's AdaOffload incumbent, round 5
  (inside the bench's timed rounds) — 256 neighbours; and a late incumbent
  (the search's incumbent at round 320, tests/golden/inc320_config3.npz),
  round 320 — 256 neighbours.
* config 4 (16 x 128): AdaOffload incumbent, round 0 — 16 neighbours.
* config 5 (32 x 256): AdaOffload incumbent, round 0 — 3 neighbours.

Seed and move mix are the bench's (bench.py SEED, MOVES).  Output:
``bench_config{N}.json.gz`` next to this script.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import multiprocessing as mp
import random
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

SEED = 20251005
MOVES = dict(shift_permille=700, max_shift=4)
FULL_TRACES = 4


def trace_digest(compute, transfers):
    """SHA-256 of the commit-ordered trace, one line per event: 'C i j k start' / 'T i j rel start'."""
    h = hashlib.sha256()
    for e in compute:
        h.update(("C %d %d %d %d\n" % tuple(e)).encode())
    for e in transfers:
        h.update(("T %d %d %d %d\n" % tuple(e)).encode())
    return h.hexdigest()


_ref = None


def _worker_init():
    global _ref
    sys.path.insert(0, REF)
    import pipesched
    _ref = pipesched


def ref_eval(numbered):
    """(k, (instance dict, orders codes [P][3m], offloaded [[i,j]], full)) -> (k, reference answers)."""
    k, job = numbered
    return k, _ref_eval(job)


def _ref_eval(job):
    ps = _ref
    inst_d, codes, off, full = job
    inst = ps.instance_from_dict(inst_d)
    F = ps.OpKind.F
    orders = {i + 1: tuple(ps.OpId(i + 1, (c >> 2) + 1, ps.OpKind(c & 3)) for c in row)
              for i, row in enumerate(codes)}
    offloaded = frozenset(ps.OpId(i, j, F) for i, j in off)
    t0 = time.perf_counter()
    out = {}
    try:
        s = ps.run_order(inst, orders, offloaded)
    except ps.OrderInfeasible as e:
        out["infeasible"] = list(e.stages)
        out["ref_seconds"] = time.perf_counter() - t0
        return out
    span = ps.makespan(s, inst)
    tr = ps.memory_trace(s, inst, ps.MemorySemantics.STRICT)
    busy = sum(inst.proc_time.values())
    comp = [[e.op.stage, e.op.microbatch, int(e.op.kind), e.start] for e in s.compute]
    trs = [[e.op.stage, e.op.microbatch, int(e.kind is ps.TransferKind.RELOAD), e.start] for e in s.transfers]
    out.update({"makespan": span, "bubble": repr(1.0 - busy / (inst.num_stages * span)),
                "peak": [tr.peak[i] for i in range(1, inst.num_stages + 1)],
                "trace_sha256": trace_digest(comp, trs), "n_compute": len(comp), "n_transfers": len(trs),
                "ref_seconds": time.perf_counter() - t0})
    if full:
        out["compute"], out["transfers"] = comp, trs
    return out


def mask_to_off(pk, mask):
    m = pk.num_microbatches
    out = []
    for b in range(pk.num_stages * m):
        if (int(mask[b >> 5]) >> (b & 31)) & 1:
            out.append([b // m + 1, b % m + 1])
    return out


def adaoffload_incumbent(inst, pk, orc):
    from paper_2510_05186_b200.heuristics import ada_backoff_sequence, filled_order
    from paper_2510_05186_b200.packing import encode_candidate
    off = frozenset(inst.offloadable_ops())
    for fills in ada_backoff_sequence(inst):
        o, mk, _ = encode_candidate(pk, {i: filled_order(inst, i, fills[i])
                                         for i in range(1, pk.num_stages + 1)}, off)
        if orc.run(o, mk)["flags"] == 1:
            return o, mk
    raise RuntimeError("no feasible AdaOffload structure")


def neighbour_set(orc, inc_o, inc_m, rnd, count, rng):
    """`count` neighbours of round `rnd` with a non-trivial move: the first count//2 such indices
    in index order, the rest drawn uniformly from the round's 65,536."""
    picked, seen = [], set()
    idx = 0
    while len(picked) < count // 2:
        t, _, _ = orc.neighbour(inc_o, inc_m, SEED, MOVES["shift_permille"], MOVES["max_shift"], rnd, idx)
        if t:
            picked.append(idx)
            seen.add(idx)
        idx += 1
    while len(picked) < count:
        idx = rng.randrange(65536)
        if idx in seen:
            continue
        t, _, _ = orc.neighbour(inc_o, inc_m, SEED, MOVES["shift_permille"], MOVES["max_shift"], rnd, idx)
        if t:
            picked.append(idx)
            seen.add(idx)
    out = []
    for idx in picked:
        t, o, mk = orc.neighbour(inc_o, inc_m, SEED, MOVES["shift_permille"], MOVES["max_shift"], rnd, idx)
        out.append((idx, t, o, mk))
    return out


def build_jobs(cfg):
    from oracle.oracle import Oracle
    from paper_2510_05186_b200 import workloads
    from paper_2510_05186_b200.instance import instance_to_dict
    from paper_2510_05186_b200.packing import pack_instance
    inst = workloads.CONFIGS[cfg]()
    pk = pack_instance(inst)
    orc = Oracle(pk)
    rng = random.Random(cfg * 1000 + 7)
    sets = []
    inc_o, inc_m = adaoffload_incumbent(inst, pk, orc)
    if cfg == 3:
        sets.append(("early", inc_o, inc_m, 5, 256))
        late = np.load(HERE / "inc320_config3.npz")
        sets.append(("late", late["orders"], late["mask"], 320, 256))
    elif cfg == 4:
        sets.append(("early", inc_o, inc_m, 0, 16))
    else:
        sets.append(("early", inc_o, inc_m, 0, 3))
    inst_d = instance_to_dict(inst)
    doc = {"config": cfg, "seed": SEED, "moves": MOVES, "instance": inst_d, "sets": []}
    jobs = []
    for name, o, mk, rnd, count in sets:
        L = 3 * pk.num_microbatches
        codes = [[int(c) for c in o[i, :L]] for i in range(pk.num_stages)]
        entry = {"name": name, "round": rnd, "incumbent": {"orders": codes, "offloaded": mask_to_off(pk, mk)},
                 "neighbours": []}
        jobs.append((entry, None, (inst_d, codes, mask_to_off(pk, mk), True)))
        for k, (idx, t, no, nmk) in enumerate(neighbour_set(orc, o, mk, rnd, count, rng)):
            diff = [[int(i), int(p), int(no[i, p])] for i, p in zip(*np.nonzero(no[:, :L] != o[:, :L]))]
            flips = [[b // pk.num_microbatches + 1, b % pk.num_microbatches + 1]
                     for b in range(pk.num_stages * pk.num_microbatches)
                     if ((int(nmk[b >> 5]) ^ int(mk[b >> 5])) >> (b & 31)) & 1]
            case = {"index": idx, "move": "shift" if t == 1 else "toggle", "order_diff": diff,
                    "offload_flips": flips}
            entry["neighbours"].append(case)
            ncodes = [[int(c) for c in no[i, :L]] for i in range(pk.num_stages)]
            jobs.append((entry, case, (inst_d, ncodes, mask_to_off(pk, nmk), k < FULL_TRACES)))
        doc["sets"].append(entry)
    return doc, jobs


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [3, 4, 5]
    todo = []
    docs = {}
    for cfg in cfgs:
        doc, jobs = build_jobs(cfg)
        docs[cfg] = doc
        todo += [(cfg, entry, case, job) for entry, case, job in jobs]
    # longest first: config 5, then 4, then 3
    todo.sort(key=lambda t: -t[0])
    t0 = time.time()
    with mp.Pool(len(__import__("os").sched_getaffinity(0)), initializer=_worker_init) as pool:
        results = pool.imap_unordered(ref_eval, list(enumerate(t[3] for t in todo)))
        pending = {cfg: sum(1 for t in todo if t[0] == cfg) for cfg in cfgs}
        for k, res in results:
            cfg, entry, case, _ = todo[k]
            (case if case is not None else entry["incumbent"]).update(res)
            pending[cfg] -= 1
            if pending[cfg] == 0:
                path = HERE / f"bench_config{cfg}.json.gz"
                with gzip.open(path, "wt") as fh:
                    json.dump(docs[cfg], fh, separators=(",", ":"))
                print(f"wrote {path} ({path.stat().st_size} bytes) at {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
