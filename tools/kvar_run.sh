timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 120 python tools/e2e_parts.py 2>&1 | tail -5
timeout 300 python bench.py --no-cpu --no-ttb 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['roofline']['simulated_events_per_launch'], d['e2e']['value'], d['e2e']['ms_per_step'])"
