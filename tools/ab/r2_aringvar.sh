#!/bin/bash
cd "$(dirname "$0")/../.."
for L in "" "$@"; do echo "== $L"
if [ -n "$L" ]; then export WL_LIB=$L; fi
timeout 300 python tools/levelbench.py --cfg 4 --ops adjoint --reps 20 | head -2
done
