timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for c in 3 2 4; do timeout 120 python tools/kvar.py $c; done
