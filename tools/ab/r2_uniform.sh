#!/bin/bash
# A/B: the analysis last-strip shift and uniform bands per kernel family (WL_UNIFORM kinds)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q > gpurun_out/uni_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/uni_pytest.log
run() { echo "== $*"; env "$@" timeout 200 python tools/opbench.py --cfg 5 --op adjoint,synthesize,residual,grad --reps 30; env "$@" timeout 100 python tools/opbench.py --cfg 4 --op adjoint,synthesize --reps 30; env "$@" timeout 100 python tools/opbench.py --cfg 3 --op adjoint,synthesize --reps 30; }
run WL_ANA_NOSHIFT=1
run WL_X=0
run WL_UNIFORM=A
run WL_UNIFORM=Aa
run WL_UNIFORM=S
run WL_UNIFORM=b
run WL_UNIFORM=R
run WL_UNIFORM=AaSsbR
for l in 1 2 3; do echo "=== anaprof level $l"; WL_LIB=ab/libwl_anaprof.so timeout 120 python tools/anaprof.py --cfg 5 --level $l | head -11; done
