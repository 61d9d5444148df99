#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_fista.py -x -q > gpurun_out/r2_multi_pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r2_multi_pytest.log
for env in "" "WL_NO_MULTI=1"; do echo "== $env"; for spec in "4 adjoint" "4 synthesize" "5 adjoint" "5 synthesize" "5 grad" "3 adjoint" "2 adjoint"; do set -- $spec; env $env timeout 120 python tools/graphbench.py --cfg $1 --op $2 --reps 30; done; done 2>&1 | tee gpurun_out/r2_multi_bench.log
