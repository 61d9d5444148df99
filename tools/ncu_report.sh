#!/bin/bash
# Text summary of ncu --set full captures: headline metrics, stall breakdown, dynamic SASS mix.
# usage: bash tools/ncu_report.sh gpurun_out/r01_prof_*.ncu-rep > profiles/r01_ncu_summary.txt
for r in "$@"; do
  echo "################ $(basename $r)"
  python "$(dirname "$0")/ncu_summary.py" "$r"
  python "$(dirname "$0")/ncu_stalls.py" "$r" | grep "stalls"
  python "$(dirname "$0")/ncu_sass_mix.py" "$r" 2>/dev/null | head -12
  echo
done
