# A/B: in-tree (with the per-candidate sync) vs the previous build
DEF=$PWD/paper_2510_05186_b200/_lib/libpipesched_b200.so
OLD=$PWD/paper_2510_05186_b200/_lib/var/libps_before.so
for rep in 1 2 3; do for L in $OLD $DEF; do for c in 5:131072 4:65536 3:65536 late3:65536 2:65536; do
  C=${c%%:*}; N=${c##*:}; INC=; if [ $C = late3 ]; then C=3; INC=tests/golden/inc320_config3.npz; fi
  KVAR_INCUMBENT=$INC PS_LIBRARY=$L timeout 300 python tools/kvar.py $C $N | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $L)', '$c', d['median_ms'])"
done; done; done
