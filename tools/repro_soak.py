"""Reproduce one tests/test_gpu_soak_random.py case step by step (diagnostics)."""
import json
import random
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402
from test_gpu_soak_random import random_tables  # noqa: E402
from paper_2510_05186_b200 import InfeasibleSchedule, NoFeasibleSchedule, instance_from_dict  # noqa: E402
from paper_2510_05186_b200.heuristics import best_feasible  # noqa: E402
from paper_2510_05186_b200.listsched import stage_order_of  # noqa: E402
from paper_2510_05186_b200.search import LocalSearch, SearchConfig  # noqa: E402

seed = int(sys.argv[1])
rng = random.Random(1000 + seed)
for _ in range(20):
    P, m = rng.randint(2, 12), rng.randint(4, 40)
    d = random_tables(rng, P, m)
    inst = instance_from_dict(d)
    try:
        s0, name = best_feasible(inst)
        torch.cuda.synchronize()
    except (InfeasibleSchedule, NoFeasibleSchedule):
        continue
    break
print("instance", P, m, name, json.dumps({k: v for k, v in d.items() if k not in ("proc_times", "mem_deltas", "act_sizes")}), flush=True)
json.dump(d, open("gpurun_out/repro_inst.json", "w"))
cfg = SearchConfig(seed=seed, neighbours=2048, shift_permille=600, max_shift=6)
ls = LocalSearch(inst, {i: stage_order_of(s0, i) for i in range(1, P + 1)}, s0.offloaded, cfg)
torch.cuda.synchronize()
print("constructed", ls.makespan, flush=True)
ms = torch.empty(2048, dtype=torch.int64, device="cuda")
for r in range(24):
    ls.launch_round(ms if r % 4 == 0 else None)
    torch.cuda.synchronize()
    ls.finish_round()
    torch.cuda.synchronize()
    print("round", r, ls.makespan, flush=True)
