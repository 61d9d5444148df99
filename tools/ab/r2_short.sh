#!/bin/bash
cd "$(dirname "$0")/../.."
for V in "" 1 6 12; do echo "== WL_SHORT_MAX=$V"
if [ -n "$V" ]; then export WL_SHORT_MAX=$V; else unset WL_SHORT_MAX; fi
timeout 300 python tools/levelbench.py --cfg 5 --ops adjoint,synthesize --reps 20
timeout 300 python tools/levelbench.py --cfg 4 --ops adjoint --reps 20
done
