# A/B timing of two libraries in one GPU call: tools/ab.sh <libA> <libB> [configs...]
A=$1; B=$2; shift 2
for c in "$@"; do
  for rep in 1 2; do
    for L in $A $B; do PS_LIBRARY=$PWD/$L timeout 120 python tools/kvar.py $c | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L'.split('/')[-1], 'cfg', d['config'], d['median_ms'], 'ms', d['cand_per_s'])"; done
  done
done
