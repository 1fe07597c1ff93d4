for n in 16384 32768 65536 131072; do KVAR_INCUMBENT=tools/inc320_config3.npz timeout 100 python tools/kvar.py 3 $n | cut -c60-200; done
