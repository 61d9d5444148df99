#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fista.py -x -q > gpurun_out/r2_a_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_a_pytest.log
for spec in "5 adjoint" "5 analyze" "5 grad" "3 adjoint" "3 analyze" "4 adjoint" "2 adjoint"; do set -- $spec; timeout 120 python tools/graphbench.py --cfg $1 --op $2 --reps 30; done 2>&1 | tee gpurun_out/r2_a_bench.log
CMD="python tools/opbench.py --cfg 5 --op adjoint --levels 1 --reps 1"; $CMD > gpurun_out/p.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ana_stream -s 3 -c 1 -o gpurun_out/r2p_ana1 -f $CMD > gpurun_out/r2p_ncu_ana.log 2>&1; echo ncu rc=$?
