#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_blur_ring.py -x -q -k "grad or ring" > gpurun_out/rf_test.log 2>&1; echo "tests rc=$?"; tail -n 2 gpurun_out/rf_test.log
for V in "" 1; do echo "== WL_NO_ROWFLAGS=$V"
if [ -n "$V" ]; then export WL_NO_ROWFLAGS=1; else unset WL_NO_ROWFLAGS; fi
for i in 1 2; do timeout 120 python tools/graphbench.py --cfg 5 --op grad --reps 40; done
done
