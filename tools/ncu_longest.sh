# Full ncu capture of the longest of the widest-grid launches of one kernel in a command (a
# batch's first pass, not a worklist pass or a few-candidate warm-start evaluation):  tools/ncu_longest.sh <kernel-regex> <out-name> <command...>
R=$1; O=$2; shift 2
ncu --clock-control none --kernel-name-base mangled -k regex:$R --metrics gpu__time_duration.sum --csv \
    --log-file gpurun_out/$O.list.csv "$@" > /dev/null 2>&1
S=$(python - gpurun_out/$O.list.csv <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
grid = lambda r: eval(r[h.index("Grid Size")].replace("(", "").replace(")", "").replace(",", "*"))
key = [(grid(r), float(r[h.index("Metric Value")].replace(",", ""))) for r in rows[1:]]
print(max(range(len(key)), key=lambda i: key[i]))
PY
)
echo "$O: longest launch index $S"
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:$R -s $S -c 1 \
    -o gpurun_out/$O -f "$@" > gpurun_out/$O.log 2>&1
