timeout 700 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
bash tools/ab.sh paper_2510_05186_b200/_lib/var/libps_prev.so paper_2510_05186_b200/_lib/libpipesched_b200.so 3
KVAR_INCUMBENT=tools/inc320_config3.npz bash tools/ab.sh paper_2510_05186_b200/_lib/var/libps_prev.so paper_2510_05186_b200/_lib/libpipesched_b200.so 3
for ks in 24 40; do echo ksmall=$ks; PS_KSMALL=$ks KVAR_INCUMBENT=tools/inc320_config3.npz timeout 100 python tools/kvar.py 3 | cut -c1-120; done
timeout 100 python tools/ttb_profile.py 3 520 | tail -1
PS_LIBRARY=$PWD/paper_2510_05186_b200/_lib/var/libps_prev.so timeout 100 python tools/ttb_profile.py 3 520 | tail -1
