#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_blur_ring.py -x -q > gpurun_out/r2_ring_pytest.log 2>&1; echo "ring pytest rc=$?"; tail -3 gpurun_out/r2_ring_pytest.log
for op in residual blur grad; do timeout 120 python tools/opbench.py --cfg 5 --op $op --reps 30; done 2>&1 | tee gpurun_out/r2_opbench.log
CMD="python tools/opbench.py --cfg 5 --op residual --reps 1"
timeout 300 $CMD > gpurun_out/r2p_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_blur_ring -s 2 -c 1 -o gpurun_out/r2p_ring -f $CMD > gpurun_out/r2p_ncu.log 2>&1; echo "ncu rc=$?"
