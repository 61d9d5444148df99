#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blur_ring.py tests/test_gpu_parity.py -x -q -k "ring or grad" > gpurun_out/par_test.log 2>&1; echo "tests rc=$?"; tail -n 1 gpurun_out/par_test.log
for L in "" build/libwl_b0.so build/libwl_b1a2.so; do echo "== $L"
if [ -n "$L" ]; then export WL_LIB=$L; fi
for i in 1 2; do timeout 300 python tools/graphbench.py --cfg 5 --op grad --reps 40; done
timeout 300 python tools/opbench.py --cfg 5 --op residual
done
