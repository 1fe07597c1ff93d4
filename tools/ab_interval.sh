# A/B of the base checkpoint interval (computes between checkpoints) per config: tools/ab_interval.sh [configs...]
for c in "$@"; do for rep in 1 2; do for iv in 8 16 32; do
  PS_CHECKPOINT_INTERVAL=$iv timeout 200 python tools/kvar.py $c $([ $c = 5 ] && echo 131072 || echo 65536) | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c interval $iv', d['median_ms'], 'ms', d['cand_per_s'])"
done; done; done
