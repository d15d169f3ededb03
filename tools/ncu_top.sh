#!/bin/bash
# ncu evidence for the dominant kernel of one cfg2 slice (M = 1024): a launch
# list of the slice (gpu__time_duration), then a full capture of the longest
# gemm_tc_persistent launch.  Usage: tools/ncu_top.sh PREC OUTDIR
set -u
PREC=${1:-tf32}; OUT=${2:-gpurun_out}
mkdir -p "$OUT"
export PREC M=1024
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file "$OUT/slice_launches_$PREC.csv" python tools/one_slice.py > "$OUT/ncu_list_$PREC.log" 2>&1
IDX=$(python - "$OUT/slice_launches_$PREC.csv" <<'PY'
import csv, sys
rows = [r for r in csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"'))]
tc = [r for r in rows if "gemm_tc_persistent" in r["Kernel Name"] and r["Metric Name"] == "gpu__time_duration.sum"]
best = max(range(len(tc)), key=lambda i: float(tc[i]["Metric Value"].replace(",", "")))
print(best)
PY
)
echo "top gemm_tc_persistent launch index: $IDX" > "$OUT/ncu_top_$PREC.txt"
ncu --profile-from-start off --set full --import-source on --clock-control none \
    --kernel-name regex:gemm_tc_persistent --launch-skip "$IDX" --launch-count 1 \
    -o "/tmp/top_$PREC" -f python tools/one_slice.py >> "$OUT/ncu_top_$PREC.txt" 2>&1
ncu -i "/tmp/top_$PREC.ncu-rep" --page raw --csv > "$OUT/top_${PREC}_raw.csv" 2>/dev/null
ncu -i "/tmp/top_$PREC.ncu-rep" --page details --csv > "$OUT/top_${PREC}_details.csv" 2>/dev/null
