# A/B of library variants on search rounds: tools/ab_libs.sh "<lib1> <lib2> ..." [configs...]
# (paths relative to the repo; "default" is the in-tree library)
LIBS=$1; shift
for c in "$@"; do for rep in 1 2; do for L in $LIBS; do
  [ $L = default ] && P=$PWD/paper_2510_05186_b200/_lib/libpipesched_b200.so || P=$PWD/$L
  PS_LIBRARY=$P timeout 200 python tools/kvar.py $c $([ $c = 5 ] && echo 131072 || echo 65536) | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c', '$L'.split('/')[-1], d['median_ms'], 'ms', d['cand_per_s'])"
done; done; done
