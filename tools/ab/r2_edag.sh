#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
for bc in symmetric symmetric_edag; do for op in adjoint synthesize analyze; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/edag_${bc}_${op}.csv python tools/bcop.py $bc $op > /dev/null 2>&1
  echo "== $bc $op"; python tools/ncu_last.py gpurun_out/edag_${bc}_${op}.csv 6
done; done
