"""CPU restatement of the search (DESIGN.md §4 descent, §4.1 iterated local search) on the C oracle.

TEST INFRASTRUCTURE: every neighbour of every round is evaluated by the oracle's restatement of
run_order, the round's best (makespan, index) key adopted on strict improvement, kicks applied
move by move with the same feasibility rule as LocalSearch.kick.  The GPU search must follow it
round for round.
"""

import numpy as np

KICK_ROUND_BASE = 1 << 40
KICK_TRIES = 64
NONE = (1 << 63) - 1


def cpu_search(orc, inc_o, inc_m, seed, permille, maxshift, n, rounds=None, kick_moves=0, kicks=None,
               patience=16, first=0, count=None):
    """Returns dict(trail=[(round, makespan, index)], best_span, best_orders, best_mask, rounds, kicks)."""
    count = n if count is None else count
    o, m = np.array(inc_o, np.uint16), np.array(inc_m, np.uint32)
    cur = int(orc.run(o, m)["makespan"])
    best = (cur, o.copy(), m.copy())
    trail, rnd, nk, stale = [], 0, 0, 0
    while True:
        if rounds is not None and rnd >= rounds:
            break
        if kicks is not None and nk >= kicks and stale >= patience:
            break
        if kick_moves > 0 and stale >= patience:
            o, m, cur = best[1].copy(), best[2].copy(), best[0]
            kept = tries = 0
            while kept < kick_moves and tries < KICK_TRIES * kick_moves:
                _, o2, m2 = orc.neighbour(o, m, seed, permille, maxshift, KICK_ROUND_BASE + nk, tries)
                tries += 1
                r = orc.run(o2, m2)
                if r["flags"] == 1:
                    kept += 1
                    o, m, cur = o2, m2, int(r["makespan"])
            nk += 1
            stale = 0
            continue
        key, _ = orc.search_round(o, m, seed, permille, maxshift, rnd, first, count)
        r = rnd
        rnd += 1
        if key != NONE and (key >> 32) < cur:
            idx = key & 0xFFFFFFFF
            _, o, m = orc.neighbour(o, m, seed, permille, maxshift, r, idx)
            cur = int(key >> 32)
            stale = 0
            if cur < best[0]:
                best = (cur, o.copy(), m.copy())
                trail.append((r, cur, idx))
        else:
            stale += 1
    return dict(trail=trail, best_span=best[0], best_orders=best[1], best_mask=best[2], rounds=rnd, kicks=nk)
