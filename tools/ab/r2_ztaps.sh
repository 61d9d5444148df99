#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_z_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_z_pytest.log
for env in "" "WL_ALL_TAPS=1"; do echo "== $env"; for spec in "5 adjoint" "5 synthesize" "5 grad" "3 adjoint" "3 synthesize" "3 analyze" "4 adjoint"; do set -- $spec; env $env timeout 120 python tools/graphbench.py --cfg $1 --op $2 --reps 30; done; done 2>&1 | tee gpurun_out/r2_z_bench.log
