python tools/base_diff.py 3 | grep -v "^ck [0-9]"
timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for rr in 0 1; do PS_REC_RESUME=$rr timeout 300 python bench.py --no-cpu --no-e2e --steps 6 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('resume', $rr, d['value'], d['ms_per_step'], d['roofline']['kernel_ms_per_launch'], d['roofline']['events_per_launch'], d['search']['final_makespan'])"; done
