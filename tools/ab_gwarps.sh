# A/B of global-state block shapes: the default library vs build/var/<variant>.so (built with
# python -m paper_2510_05186_b200.build -DPS_GSTATE_MAX_WARPS=W -DPS_MIN_BLOCKS_G=B --out=build/var/<variant>.so)
#   tools/ab_gwarps.sh <variant> [configs...]
V=$1; shift
for c in "$@"; do for rep in 1 2; do for L in paper_2510_05186_b200/_lib/libpipesched_b200.so build/var/$V.so; do
  PS_LIBRARY=$PWD/$L timeout 200 python tools/kvar.py $c $([ $c = 5 ] && echo 131072 || echo 65536) | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg $c', '$L'.split('/')[-1], d['median_ms'], 'ms', d['cand_per_s'])"
done; done; done
