# compute-sanitizer memcheck over a few random-instance soak cases of each path (odd shapes,
# shared channels, 64-bit ledgers): any invalid access or leak report fails the line.
O=gpurun_out
run() { timeout 900 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python tools/soak_random.py "$@" > $O/san_$1_$4.log 2>&1; echo "$* rc=$? $(grep -c 'Invalid\|misaligned' $O/san_$1_$4.log) errors"; }
run 0 8 small search
run 500 4 big search
run 2000 6 small channel
run 2500 3 big channel
run 3000 6 small batch
run 3500 4 big batch
# shared-memory hazards and barrier use on odd layouts (slow: two cases each)
for tool in racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 10 --error-exitcode 9 python tools/soak_random.py 1 2 small search > $O/san_${tool}_search.log 2>&1; echo "$tool search rc=$? $(tail -1 $O/san_${tool}_search.log)"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 10 --error-exitcode 9 python tools/soak_random.py 2001 2 small channel > $O/san_${tool}_channel.log 2>&1; echo "$tool channel rc=$? $(tail -1 $O/san_${tool}_channel.log)"
  timeout 1200 compute-sanitizer --tool $tool --print-limit 10 --error-exitcode 9 python tools/soak_random.py 3001 2 big batch > $O/san_${tool}_batch.log 2>&1; echo "$tool batch rc=$? $(tail -1 $O/san_${tool}_batch.log)"
done
