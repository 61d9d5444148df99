#!/bin/bash
# ring blur A/B: parity + residual / blur / grad timings (+ WL_LIB variants given as args)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_blur_ring.py -x -q > gpurun_out/ring_test.log 2>&1; echo "ring tests rc=$?"; tail -2 gpurun_out/ring_test.log
timeout 300 python tools/opbench.py --cfg 5 --op residual,blur,grad
for L in "$@"; do echo "== $L"; WL_LIB=$L timeout 300 python tools/opbench.py --cfg 5 --op residual,blur; done
WL_LIB=build/libwl_prof.so timeout 300 python tools/ringprof.py
