#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_test.log 2>&1; echo "gpu tests rc=$?"; tail -n 3 gpurun_out/gpu_test.log
for V in "" 1; do echo "== WL_NO_TAIL=$V"
if [ -n "$V" ]; then export WL_NO_TAIL=1; else unset WL_NO_TAIL; fi
timeout 300 python tools/levelbench.py --cfg 4 --ops adjoint,analyze --reps 20
timeout 300 python tools/levelbench.py --cfg 5 --ops adjoint --reps 20
for c in 1 2 3; do timeout 300 python tools/graphbench.py --cfg $c --op adjoint --reps 30; done
timeout 300 python tools/opbench.py --cfg 5 --op grad
done
