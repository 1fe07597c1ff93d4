timeout 700 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 100 python tools/ttb_profile.py 3 520 | tail -1
python -c "
import sys; sys.path.insert(0,'.')
import time
from paper_2510_05186_b200 import workloads
from paper_2510_05186_b200.search import SearchConfig, warm_start_search
inst = workloads.CONFIGS[3]()
for dd in (True, False):
    t=time.perf_counter(); r = warm_start_search(inst, SearchConfig(seed=20251005, neighbours=65536, shift_permille=700, max_shift=4, dedup=dd), rounds=2000, patience=16)
    print('dedup', dd, 'rounds', r.rounds, 'best', r.makespan, 'elapsed', round(r.elapsed,3), 'to best', round(r.improvements[-1].timestamp,3))
"
