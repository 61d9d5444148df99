#!/bin/bash
# ring analysis A/B: parity + per-level chain timings (WL_NO_ARING set = streaming kernel)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fista.py tests/test_gpu_graph.py -x -q > gpurun_out/par_test.log 2>&1; echo "parity tests rc=$?"; tail -3 gpurun_out/par_test.log
run() {
timeout 300 python tools/levelbench.py --cfg 4 --ops adjoint --reps 20
timeout 300 python tools/levelbench.py --cfg 5 --ops adjoint --reps 20
timeout 300 python tools/opbench.py --cfg 5 --op grad
timeout 300 python tools/opbench.py --cfg 3 --op adjoint
timeout 300 python tools/opbench.py --cfg 2 --op adjoint
}
echo "== ring"; run
echo "== stream"; export WL_NO_ARING=1; run
