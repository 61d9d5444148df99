#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "not native_library" > gpurun_out/r2_e_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2_e_pytest.log
timeout 300 python tools/bcbench.py 2>&1 | tee gpurun_out/r2_bcbench.log

