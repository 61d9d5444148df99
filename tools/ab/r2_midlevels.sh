#!/bin/bash
# ncu --set full of every level kernel of one cfg5 W* chain and one W chain (mid-level overheads)
cd "$(dirname "$0")/../.."
for op in adjoint synthesize; do
  C="python tools/opbench.py --cfg 5 --op $op --reps 1"
  timeout 300 $C > /dev/null 2>&1 || { echo "plain $op failed"; continue; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_ana_stream|k_synth_stream' -c 10 \
    -o gpurun_out/mid_$op -f $C > gpurun_out/mid_$op.log 2>&1; echo "ncu $op rc=$?"
done
