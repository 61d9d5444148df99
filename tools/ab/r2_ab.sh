#!/bin/bash
# A/B of ab/*.so builds on the cfg5 blur ops (usage: bash tools/r2_ab.sh "ops" lib...)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
OPS=${1:-residual,blur}; shift
for L in paper_1707_02018_b200/libwl.so "$@"; do echo "== $L"; WL_LIB=$L timeout 120 python tools/opbench.py --cfg 5 --op $OPS --reps 30; done 2>&1 | tee gpurun_out/r2_ab.log
