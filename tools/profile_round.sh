#!/bin/bash
# Round-end evidence on one GPU (under gpurun): bench line, ncu launch list of the bench step,
# and one `ncu --set full` capture per hot kernel (each command first runs clean without ncu).
# usage: bash tools/profile_round.sh <tag>      -> gpurun_out/<tag>_*
cd "$(dirname "$0")/.."
T=${1:-r01}
O=gpurun_out
mkdir -p $O
timeout 600 python bench.py --steps 20 --warmup 5 > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $CMD > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $O/${T}_launches.csv $CMD > $O/${T}_ncu_launches.log 2>&1; echo "launches rc=$?"
full() {  # name regex command...
  local name=$1 re=$2; shift 2
  timeout 300 "$@" > /dev/null 2>&1 || { echo "$name: plain run failed"; return; }
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$re -s 3 -c 1 -o $O/${T}_prof_$name -f "$@" \
    > $O/${T}_ncu_$name.log 2>&1; echo "ncu $name rc=$?"
}
full blur_residual k_blur_stream python tools/opbench.py --cfg 5 --op residual --reps 2
full ana_l1 k_ana_stream python tools/opbench.py --cfg 5 --op adjoint --levels 1 --reps 2
full syn_l1 k_synth_stream python tools/opbench.py --cfg 5 --op synthesize --levels 1 --reps 2
full fista_ana_l1 k_ana_stream python tools/opbench.py --cfg 5 --op fista --levels 1 --reps 2
full ana_l1_cfg4 k_ana_stream python tools/opbench.py --cfg 4 --op adjoint --levels 1 --reps 2
full bce_grad k_bce_grad python tools/bcebench.py --problems 4096 --reps 2
