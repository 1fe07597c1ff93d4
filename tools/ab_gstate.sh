# A/B of the global-state kernel build: tools/ab_gstate.sh (needs build/var/g3.so, g4.so from
#   python -m paper_2510_05186_b200.build -DPS_MIN_BLOCKS_G=N --out=build/var/gN.so)
for rep in 1 2; do
for v in "default 1" "default 4" "build/var/g3.so 4" "build/var/g4.so 4"; do
  set -- $v
  if [ $1 = default ]; then L=$PWD/paper_2510_05186_b200/_lib/libpipesched_b200.so; else L=$PWD/$1; fi
  PS_GSTATE_WARPS=$2 PS_LIBRARY=$L timeout 200 python tools/kvar.py 5 131072 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 warps=$2', d['median_ms'], 'ms', d['cand_per_s'])"
done; done
