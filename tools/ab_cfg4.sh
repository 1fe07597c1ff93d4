# A/B of the occupancy-driven global-state rule: search rounds (kvar) and the e2e host path (bench).
for rep in 1 2; do for t in 0 12; do
  PS_GSTATE_BELOW_WARPS=$t timeout 200 python tools/kvar.py 4 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 below=$t', d['median_ms'], 'ms', d['cand_per_s'])"
done; done
for g in 0 1; do
  PS_GSTATE_RULE=$g timeout 300 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu --no-ttb 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 bench gstate_rule=$g value', d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'])"
done
