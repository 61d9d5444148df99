#!/bin/bash
# A/B: register caps (launch bounds) of the level kernels and the ring blur; usage: r2_regcap.sh lib...
cd "$(dirname "$0")/../.."
for L in "$@"; do echo "== $L"
  WL_LIB=$L timeout 200 python tools/opbench.py --cfg 5 --op adjoint,synthesize,residual,grad --reps 30
  WL_LIB=$L timeout 100 python tools/opbench.py --cfg 3 --op adjoint,synthesize --reps 30
  WL_LIB=$L timeout 100 python tools/opbench.py --cfg 4 --op adjoint,synthesize --reps 30
done
