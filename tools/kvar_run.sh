timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for c in 3 2 4; do timeout 120 python tools/kvar.py $c; done
KVAR_INCUMBENT=tools/inc320_config3.npz timeout 100 python tools/kvar.py 3
