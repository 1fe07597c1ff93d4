O=gpurun_out
timeout 600 python tools/soak_random.py 2000 100 small channel > $O/soak_ch_small.jsonl 2>&1; tail -1 $O/soak_ch_small.jsonl
timeout 400 python tools/soak_random.py 2500 20 big channel > $O/soak_ch_big.jsonl 2>&1; tail -1 $O/soak_ch_big.jsonl
timeout 400 python tools/soak_random.py 2700 8 wide channel > $O/soak_ch_wide.jsonl 2>&1; tail -1 $O/soak_ch_wide.jsonl
timeout 500 python tools/soak_random.py 3000 100 small batch > $O/soak_b_small.jsonl 2>&1; tail -1 $O/soak_b_small.jsonl
timeout 400 python tools/soak_random.py 3500 30 big batch > $O/soak_b_big.jsonl 2>&1; tail -1 $O/soak_b_big.jsonl
timeout 400 python tools/soak_random.py 3700 10 wide batch > $O/soak_b_wide.jsonl 2>&1; tail -1 $O/soak_b_wide.jsonl
