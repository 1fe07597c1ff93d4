for rep in 1 2; do
for e in "PS_WIN_SMEM=0" "PS_WIN_SMEM=1"; do
  for c in "5 131072" "4 65536"; do
    env $e timeout 300 python tools/kvar.py $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', '$c', d['median_ms'], 'ms', d['cand_per_s'])"
  done
done; done
