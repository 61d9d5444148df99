#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blur_ring.py -x -q > gpurun_out/r2_ring_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_ring_pytest.log
for L in paper_1707_02018_b200/libwl.so ab/libwl_R2M4.so; do echo "== $L"; WL_LIB=$L timeout 120 python tools/opbench.py --cfg 5 --op residual,grad --reps 30; done
echo "== ring2 off"; WL_RING2_OFF=1 timeout 120 python tools/opbench.py --cfg 5 --op residual --reps 30
