# A/B of library builds on search rounds: tools/ab_lib.sh <variant.so>... (each against the in-tree
# library; configs 5, 4, 3 and the late config-3 incumbent; two passes to expose noise)
DEF=$PWD/paper_2510_05186_b200/_lib/libpipesched_b200.so
LIBS="$DEF $*"
CFGS=${AB_CONFIGS:-"5:131072 4:65536 3:65536 late3:65536"}
for rep in 1 2; do
for L in $LIBS; do
  for c in $CFGS; do
    C=${c%%:*}; N=${c##*:}; INC=
    if [ $C = late3 ]; then C=3; INC=tests/golden/inc320_config3.npz; fi
    KVAR_INCUMBENT=$INC PS_LIBRARY=$L timeout 300 python tools/kvar.py $C $N | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $L)', '$c', d['median_ms'], 'ms', d['cand_per_s'])"
  done
done; done
