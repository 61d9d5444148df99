#!/bin/bash
# round-2 probe: pipe microbench, per-level marginal costs, residual/blur timings
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench/pipes.cu -o /tmp/pipes && timeout 60 /tmp/pipes > gpurun_out/pipes.log 2>&1; echo "pipes rc=$?"
cat gpurun_out/pipes.log
timeout 300 python tools/levelbench.py --cfg 4 --ops adjoint,synthesize > gpurun_out/levels_cfg4.log 2>&1; echo "lv4 rc=$?"
cat gpurun_out/levels_cfg4.log
timeout 300 python tools/levelbench.py --cfg 5 --ops adjoint,synthesize --reps 20 > gpurun_out/levels_cfg5.log 2>&1; echo "lv5 rc=$?"
cat gpurun_out/levels_cfg5.log
timeout 300 python tools/opbench.py --cfg 5 --op residual,blur,grad > gpurun_out/op5.log 2>&1; echo "op5 rc=$?"
cat gpurun_out/op5.log
