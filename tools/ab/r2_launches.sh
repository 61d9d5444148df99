#!/bin/bash
# launch lists: cfg5 grad step, cfg4 W* chain (with DRAM bytes), cfg5 W / W* chains
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for spec in "5 grad" "4 adjoint" "5 adjoint" "5 synthesize" "4 synthesize"; do
  set -- $spec
  CMD="python tools/opbench.py --cfg $1 --op $2 --reps 1"
  timeout 300 $CMD > /dev/null 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r2_launch_cfg$1_$2.csv $CMD > /dev/null 2>&1; echo "cfg$1 $2 rc=$?"
done
for spec in "5 adjoint" "5 synthesize" "4 adjoint" "4 synthesize" "5 grad"; do set -- $spec; timeout 120 python tools/graphbench.py --cfg $1 --op $2 --reps 30; done 2>&1 | tee gpurun_out/r2_graphbench.log
