# A/B: shared-memory state vs global-scratch state (PS_FORCE_GSTATE) per config, one GPU call.
#   tools/ab_force_g.sh [configs...]
for c in "$@"; do for rep in 1 2; do for g in 0 1; do
  PS_FORCE_GSTATE=$g timeout 200 python tools/kvar.py $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c gstate=$g', d['median_ms'], 'ms', d['cand_per_s'])"
done; done; done
for g in 0 1; do
  KVAR_INCUMBENT=tests/golden/inc320_config3.npz PS_FORCE_GSTATE=$g timeout 200 python tools/kvar.py 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('late cfg3 gstate=$g', d['median_ms'], 'ms', d['cand_per_s'])"
done
