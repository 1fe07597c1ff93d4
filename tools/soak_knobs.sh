# Random-instance soaks under the planner's alternative launch plans (env knobs of ps_abi.cu):
# global-state kernels, windows in global memory, tiny ledger windows (overflow hand-over to a
# wider pass), other checkpoint intervals, no word masks, no no-base build, static distribution.
O=gpurun_out
for knobs in "PS_FORCE_GSTATE=1" "PS_FORCE_GSTATE=1 PS_WIN_SMEM=0" "PS_WINDOW=4" "PS_CHECKPOINT_INTERVAL=1" \
             "PS_CHECKPOINT_INTERVAL=32" "PS_WMASK=0 PS_FORCE_GSTATE=1" "PS_NOBASE_BUILD=0" "PS_DYNAMIC=0 PS_ORDER=0" \
             "PS_FORCE_GSTATE=1 PS_GSTATE_WARPS=1" "PS_SEARCH_ROWS=1"; do
  tag=$(echo $knobs | tr ' =' '_-')
  for path in "search 5000 30" "channel 5100 20" "batch 5200 20"; do
    set -- $path
    env $knobs timeout 600 python tools/soak_random.py $2 $3 small $1 > $O/knob_${tag}_$1.jsonl 2>&1
    echo "$knobs $1 rc=$? $(tail -1 $O/knob_${tag}_$1.jsonl | cut -c1-150)"
  done
done
