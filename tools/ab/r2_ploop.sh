#!/bin/bash
# A/B: the prologue of the 4-stage level kernels as a loop (one copy of the block loader instead of NS-1)
cd "$(dirname "$0")/../.."
for L in paper_1707_02018_b200/libwl.so ab/libwl_ploop.so; do echo "== $L"
  for c in 5 4 3 2; do WL_LIB=$L timeout 100 python tools/graphbench.py --cfg $c --op adjoint --reps 40 | tail -1; WL_LIB=$L timeout 100 python tools/graphbench.py --cfg $c --op synthesize --reps 40 | tail -1; done
  WL_LIB=$L timeout 100 python tools/graphbench.py --cfg 5 --op grad --reps 40 | tail -1
done
