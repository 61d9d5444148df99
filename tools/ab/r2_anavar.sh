#!/bin/bash
# analysis tile / stage A/B (WL_LIB variants given as args): cfg5 and cfg4 W* level timings
cd "$(dirname "$0")/../.."
for L in "" "$@"; do echo "== $L"
if [ -n "$L" ]; then export WL_LIB=$L; fi
timeout 300 python tools/levelbench.py --cfg 5 --ops adjoint --reps 20 | head -2
timeout 300 python tools/levelbench.py --cfg 4 --ops adjoint --reps 20 | sed -n '6p'
timeout 300 python tools/opbench.py --cfg 3 --op adjoint,analyze
done
