#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
WL_LIB=build/libwl_nb4.so timeout 600 python -m pytest tests/test_gpu_blur_ring.py tests/test_gpu_parity.py -x -q -k "ring or grad or blur" > gpurun_out/ring_test.log 2>&1; echo "nb4 ring tests rc=$?"; tail -n 1 gpurun_out/ring_test.log
timeout 300 python tools/opbench.py --cfg 5 --op residual,blur,grad
WL_LIB=build/libwl_nb4.so timeout 300 python tools/opbench.py --cfg 5 --op residual,blur,grad
