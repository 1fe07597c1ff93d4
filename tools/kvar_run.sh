for bps in 2 8 16; do PS_FORCE_GSTATE=1 PS_GSTATE_BLOCKS_PER_SM=$bps timeout 300 python tools/kvar.py 5 16384 2>&1 | tail -1; done
for bps in 8 16; do PS_FORCE_GSTATE=1 PS_GSTATE_BLOCKS_PER_SM=$bps timeout 300 python tools/kvar.py 4 65536 2>&1 | tail -1; done
