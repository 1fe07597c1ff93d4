# Base-recording times per library build: tools/rec_ab.sh <variant.so>... (against the in-tree one)
for L in $PWD/paper_2510_05186_b200/_lib/libpipesched_b200.so "$@"; do
for c in "5 131072 8" "4 65536 10" "3 65536 20"; do
PS_LIBRARY=$L timeout 600 python tools/rec_time.py $c | sed "s|^|$(basename $L) |"
done; done
