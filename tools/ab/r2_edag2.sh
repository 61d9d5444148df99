#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fista.py -x -q > gpurun_out/par_test.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/par_test.log
timeout 300 python tools/bcbench.py
for bc in symmetric symmetric_edag; do for op in adjoint analyze; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/edag_${bc}_${op}.csv python tools/bcop.py $bc $op > /dev/null 2>&1
  echo "== $bc $op"; python tools/ncu_last.py gpurun_out/edag_${bc}_${op}.csv 5
done; done
