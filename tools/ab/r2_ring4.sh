#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blur_ring.py tests/test_gpu_parity.py -x -q -k "ring or blur or grad" > gpurun_out/r2_ring_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_ring_pytest.log
bash tools/r2_ab.sh residual,blur,grad ab/libwl_nofix.so
