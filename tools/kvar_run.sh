PS_LIBRARY=$PWD/paper_2510_05186_b200/_lib/var/libps_dbgev.so timeout 300 python tools/event_stats.py 3 2>&1 | head -4
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 120 python tools/kvar.py 3
