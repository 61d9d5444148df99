#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/par_test.log 2>&1; echo "parity rc=$?"; tail -n 1 gpurun_out/par_test.log
for L in "" build/libwl_h0.so build/libwl_h2.so; do echo "== $L"
if [ -n "$L" ]; then export WL_LIB=$L; fi
timeout 300 python tools/levelbench.py --cfg 5 --ops adjoint,synthesize --reps 20
timeout 300 python tools/levelbench.py --cfg 4 --ops adjoint --reps 20 | tail -1
timeout 300 python tools/graphbench.py --cfg 5 --op grad --reps 30
done
