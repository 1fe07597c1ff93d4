timeout 700 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash tools/ab.sh paper_2510_05186_b200/_lib/var/libps_prev.so paper_2510_05186_b200/_lib/libpipesched_b200.so 3 2 4
KVAR_INCUMBENT=tools/inc320_config3.npz bash tools/ab.sh paper_2510_05186_b200/_lib/var/libps_prev.so paper_2510_05186_b200/_lib/libpipesched_b200.so 3
