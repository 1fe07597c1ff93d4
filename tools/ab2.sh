# A/B of two library variants in one GPU call: search rounds (kvar.py) on configs 3/2/4, the
# late config-3 incumbent, and the materialised host path (bench.py e2e) on config 3.
#   tools/ab2.sh <libA> <libB>
A=$1; B=$2
kv() { PS_LIBRARY=$PWD/$1 timeout 120 python tools/kvar.py $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1'.split('/')[-1], 'cfg', d['config'], '$3', d['median_ms'], 'ms', d['cand_per_s'])"; }
for c in 3 2 4; do for rep in 1 2; do kv $A $c; kv $B $c; done; done
for rep in 1 2; do KVAR_INCUMBENT=tools/inc320_config3.npz kv $A 3 late; KVAR_INCUMBENT=tools/inc320_config3.npz kv $B 3 late; done
for rep in 1 2; do for L in $A $B; do PS_LIBRARY=$PWD/$L timeout 300 python bench.py --config 3 --no-cpu --no-ttb --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L'.split('/')[-1], 'bench3', round(d['value']), 'e2e', round(d['e2e']['value']))"; done; done
