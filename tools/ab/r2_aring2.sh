#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "adjoint or grad or analy" > gpurun_out/par_test.log 2>&1; echo "parity tests rc=$?"; tail -1 gpurun_out/par_test.log
for L in "" build/libwl_s4.so; do echo "== $L"
if [ -n "$L" ]; then export WL_LIB=$L; fi
timeout 300 python tools/levelbench.py --cfg 4 --ops adjoint --reps 20
timeout 300 python tools/levelbench.py --cfg 5 --ops adjoint --reps 20
done
