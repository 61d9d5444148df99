#!/bin/bash
# A/B: register caps (launch bounds) of the level kernels
cd "$(dirname "$0")/../.."
for L in paper_1707_02018_b200/libwl.so ab/libwl_a512.so ab/libwl_a640.so ab/libwl_s1024.so; do echo "== $L"
  WL_LIB=$L timeout 200 python tools/opbench.py --cfg 5 --op adjoint,synthesize,grad --reps 30
  WL_LIB=$L timeout 100 python tools/opbench.py --cfg 3 --op adjoint,synthesize --reps 30
  WL_LIB=$L timeout 100 python tools/opbench.py --cfg 4 --op adjoint,synthesize --reps 30
done
