#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
WL_ARING=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fista.py -x -q > gpurun_out/par_test.log 2>&1; echo "parity (forced ring) rc=$?"; tail -n 1 gpurun_out/par_test.log
for A in 1 ""; do echo "== WL_ARING=$A"
if [ -n "$A" ]; then export WL_ARING=1; else unset WL_ARING; fi
timeout 300 python tools/levelbench.py --cfg 4 --ops adjoint --reps 20
timeout 300 python tools/levelbench.py --cfg 5 --ops adjoint --reps 20
timeout 300 python tools/opbench.py --cfg 3 --op adjoint
done
