#!/bin/bash
# A/B: the compact instantiations of the level kernels (WL_NO_PLAIN=1: the general ones)
cd "$(dirname "$0")/../.."
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/plain_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/plain_pytest.log
for e in WL_NO_PLAIN=1 WL_X=0; do echo "== $e"
  for c in 5 4 3 2; do env $e timeout 100 python tools/graphbench.py --cfg $c --op adjoint --reps 40 | tail -1; env $e timeout 100 python tools/graphbench.py --cfg $c --op synthesize --reps 40 | tail -1; done
  env $e timeout 100 python tools/graphbench.py --cfg 5 --op grad --reps 40 | tail -1
done
