#!/bin/bash
# One GPU session: parity tests, smoke, microbench, bench, ncu launch list + full capture of the top kernel.
# usage (under gpurun): bash tools/gpu_check.sh [kernel-regex[,kernel-regex...]]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
K=${1:-blur_residual}
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_gpu rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
if [ -n "$MICRO" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/microbench/ffma.cu -o /tmp/ffma && timeout 120 /tmp/ffma > gpurun_out/ffma.log 2>&1; echo "ffma rc=$?"
fi
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
if [ -z "$NONCU" ]; then
  timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
  for KK in $(echo $K | tr ',' ' '); do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KK -s 2 -c 1 -o gpurun_out/prof_$KK -f $CMD > gpurun_out/ncu_full_$KK.log 2>&1; echo "ncu full $KK rc=$?"
  done
fi
