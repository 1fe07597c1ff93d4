timeout 300 python tools/prefix_diff.py 4 2>&1 | tail -1
NCAND=256 REPS=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool initcheck --print-limit 3 python tools/prefix_diff.py 2 > gpurun_out/initcheck.txt 2>&1; grep -A3 "Uninit" gpurun_out/initcheck.txt | head -12; grep "SUMMARY" gpurun_out/initcheck.txt
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
