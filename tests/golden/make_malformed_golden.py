"""Reference outcomes for malformed stage orders (rows that are not permutations of the stage's ops).

Run here (the reference is importable only in the build container):

    python tests/golden/make_malformed_golden.py

``run_order`` (listsched.py:167-269) does not validate its input: it replays every row literally —
a repeated op is committed again, a short row simply ends — and since some op of a malformed row
is never committed it ends in ``OrderInfeasible`` whose ``stages`` are the rows not yet exhausted
when no event can start (listsched.py:248-252).  This records, with the unmodified reference,
that outcome for rows with a repeated op (damage early, in the middle and in the last stage),
rows missing an op, and short rows, over derived and explicit channel modes.
Output: ``malformed.json.gz`` next to this script.
"""

from __future__ import annotations

import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from make_golden import base_structures, dump, perturb, ps, record, to_ref  # noqa: E402
from paper_2510_05186_b200 import workloads  # noqa: E402


def damaged(inst, orders, rng, how, stage):
    new = {i: list(orders[i]) for i in orders}
    row = new[stage]
    if how == "repeat":                 # an op replaced by a copy of another op of the same row
        a, b = rng.sample(range(len(row)), 2)
        row[a] = row[b]
    elif how == "missing":              # an op removed (row one shorter)
        del row[rng.randrange(len(row))]
    elif how == "short":                # the row's tail cut off
        del row[rng.randint(1, len(row) - 1):]
    elif how == "empty":
        row.clear()
    return {i: tuple(v) for i, v in new.items()}


def main():
    rng = random.Random(77)
    insts = [ps.make_uniform_instance(*a) for a in [(2, 3, 1, 1, 1, 1, 1, 2, 3), (4, 6, 1, 1, 1, 0, 1, 2, 3),
                                                     (3, 4, 1, 1, 1, 1, 1, 2, 8), (4, 8, 2, 2, 1, 1, 1, 2, 8)]]
    insts += [ps.random_instance(s, 3, 3, mem_profile="tight") for s in range(3)]
    insts += [to_ref(workloads.config2())]
    out = []
    for inst in insts:
        P = inst.num_stages
        entry = {"instance": ps.instance_to_dict(inst), "cases": []}
        structs = base_structures(inst)
        for k in range(24 if P <= 4 else 12):
            o, f = structs[rng.randrange(len(structs))]
            if rng.random() < 0.5:
                o, f = perturb(inst, o, f, rng, rng.randint(0, 2), 0.0)
            how = ("repeat", "missing", "short", "empty")[k % 4]
            stage = (1, P, rng.randint(1, P))[k % 3]
            bad = damaged(inst, o, rng, how, stage)
            c, s = record(inst, bad, f)
            c["damage"] = [how, stage]
            entry["cases"].append(c)
            if k % 3 == 0 and s is None and len(inst.topology_groups) and f:
                # explicit channel mode: the damaged rows with the channel orders of the intact ones
                try:
                    good = ps.run_order(inst, o, f)
                except ps.OrderInfeasible:
                    continue
                co = {g: ps.channel_order_of(good, inst, g) for g in range(len(inst.topology_groups))}
                c2, _ = record(inst, bad, f, co)
                c2["damage"] = [how, stage]
                entry["cases"].append(c2)
        out.append(entry)
    dump({"name": "malformed", "instances": out}, "malformed.json.gz")


if __name__ == "__main__":
    main()
