# Checkpoint interval (compute events between checkpoints) on early and late config-3 rounds.
for rep in 1 2; do for iv in 4 8 16; do
  for inc in "" tests/golden/inc320_config3.npz; do
    PS_CHECKPOINT_INTERVAL=$iv KVAR_INCUMBENT=$inc timeout 300 python tools/kvar.py 3 65536 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('interval $iv', 'late' if '$inc' else 'early', d['median_ms'], 'ms', d['events_last'])"
  done
done; done
