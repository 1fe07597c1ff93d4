# Early vs late config-3 search rounds by move mix, then with the search's dedup and bound pruning.
run() { timeout 200 python tools/kvar.py 3 65536 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['shift_permille'], 'dedup', d['dedup'], 'cutoff', d['cutoff'], d['median_ms'], 'ms', d['events_last'], d['events_full'])"; }
for inc in "" tests/golden/inc320_config3.npz; do
  tag=$([ -n "$inc" ] && echo late || echo early)
  for sp in 700 1000 0; do KVAR_SHIFT=$sp KVAR_INCUMBENT=$inc run $tag; done
  KVAR_DEDUP=1 KVAR_INCUMBENT=$inc run $tag
  KVAR_DEDUP=1 KVAR_PRUNE=1 KVAR_INCUMBENT=$inc run $tag
done
