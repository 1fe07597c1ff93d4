# Round-end refresh on the GPU box: the GPU suite, bench lines for every BASELINE config, the launch
# list of the default bench command and ncu --set full captures of the evaluator's main launches.
#   bash tools/refresh.sh <tag>      (outputs under gpurun_out/<tag>_*)
T=${1:-rf}
O=gpurun_out
python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/${T}_gputest.log 2>&1; echo "gpu tests rc=$?"; tail -2 $O/${T}_gputest.log
python bench.py > $O/${T}_bench_c3.json 2> $O/${T}_bench_c3.err; echo "bench c3 rc=$?"
python bench.py --config 5 --per-gpu 131072 --steps 10 > $O/${T}_bench_c5.json 2> $O/${T}_bench_c5.err; echo "bench c5 rc=$?"
python bench.py --config 4 --per-gpu 16384 --steps 20 --ttb-rounds 400 > $O/${T}_bench_c4_16384.json 2> $O/${T}_bench_c4.err; echo "bench c4 rc=$?"
python bench.py --config 2 --per-gpu 4096 --steps 30 > $O/${T}_bench_c2_4096.json 2> $O/${T}_bench_c2.err; echo "bench c2 rc=$?"
python bench.py --config 1 --per-gpu 4096 --steps 30 > $O/${T}_bench_c1_4096.json 2> $O/${T}_bench_c1.err; echo "bench c1 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${T}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-ttb --no-cpu > /dev/null 2>&1; echo "launch list rc=$?"
bash tools/ncu_longest.sh IiLb1ELi0ELb0ELb1ELb1E ${T}_early python tools/kvar.py 3 65536
KVAR_INCUMBENT=tests/golden/inc320_config3.npz bash tools/ncu_longest.sh IiLb1ELi0ELb0ELb1ELb1E ${T}_late python tools/kvar.py 3 65536
bash tools/ncu_longest.sh IiLb1ELi2ELb0ELb1ELb1E ${T}_cfg5 python tools/kvar.py 5 131072
bash tools/ncu_longest.sh IiLb1ELi1ELb0ELb1ELb1E ${T}_cfg4 python tools/kvar.py 4 65536
ls -la $O | tail -30
