#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_test.log 2>&1; echo "gpu tests rc=$?"; tail -n 3 gpurun_out/gpu_test.log
for V in "" 1; do echo "== WL_NO_SMALL=$V"
if [ -n "$V" ]; then export WL_NO_SMALL=1; else unset WL_NO_SMALL; fi
for c in 1 2 3 4 5; do timeout 300 python tools/graphbench.py --cfg $c --op adjoint --reps 30; timeout 300 python tools/graphbench.py --cfg $c --op synthesize --reps 30; done
done
