PS_LIBRARY=$PWD/paper_2510_05186_b200/_lib/var/libps_dbgconv.so timeout 300 python tools/conv_stats.py 3 2>&1 | tail -9
