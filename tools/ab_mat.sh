# A/B of library builds on materialised batches: tools/ab_mat.sh <variant.so>...
for rep in 1 2; do
for L in $PWD/paper_2510_05186_b200/_lib/libpipesched_b200.so "$@"; do
  for c in ${AB_CONFIGS:-3 2 4}; do PS_LIBRARY=$L timeout 300 python tools/mat_time.py $c; done
done; done
