#!/bin/bash
# per-kernel SM busy-time spread of one cfg5 grad step and one cfg4 W* chain (how much a static run partition leaves idle)
cd "$(dirname "$0")/../.."
M=gpu__time_duration.sum,sm__cycles_active.min,sm__cycles_active.max,sm__cycles_active.avg,sm__cycles_elapsed.max
for spec in "5 grad" "4 adjoint"; do
  set -- $spec
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/spread_cfg$1_$2.csv \
    python tools/opbench.py --cfg $1 --op $2 --reps 1 > /dev/null 2>&1; echo "spread cfg$1 $2 rc=$?"
done
