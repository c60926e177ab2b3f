#!/bin/bash
# Dev tool: per-kernel device durations of the single-frame pipeline (ncu, serialized).
# usage (on the GPU box): tools/kernel_times.sh [chip]
chip=${1:-1}
python tools/run_frame.py $chip 3 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"scan_kernel|value_kernel" -s 4 -c 4 --csv python tools/run_frame.py $chip 3 2>/dev/null | \
  python3 -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10 and r[0].isdigit()]
for r in rows: print(r[4][:40].ljust(42), r[-1], 'ns')
"
