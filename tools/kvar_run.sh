timeout 60 python tools/ttb_profile.py 3 40 2>&1 | tail -2; echo "ttb rc=$?"
timeout 700 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().split('\n')[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['cpu_baseline']['parity'], d['time_to_best']['seconds_to_best'], d['clocks'])"
