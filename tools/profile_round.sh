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
full blur_residual k_blur_ring python tools/opbench.py --cfg 5 --op residual --reps 2
full ana_l1 k_ana_stream python tools/opbench.py --cfg 5 --op adjoint --levels 1 --reps 2
full syn_l1 k_synth_stream python tools/opbench.py --cfg 5 --op synthesize --levels 1 --reps 2
full fista_ana_l1 k_ana_stream python tools/opbench.py --cfg 5 --op fista --levels 1 --reps 2
full ana_l1_cfg4 k_ana_ring python tools/opbench.py --cfg 4 --op adjoint --levels 1 --reps 2
full bce_grad k_bce_grad python tools/bcebench.py --problems 4096 --reps 2
# per-launch DRAM bytes: one cfg5 grad step, one cfg4 W* chain, one cfg3-shape EDAG W and W*
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for spec in "5 grad" "4 adjoint"; do
  set -- $spec
  C2="python tools/opbench.py --cfg $1 --op $2 --reps 1"
  timeout 300 $C2 > /dev/null 2>&1 && timeout 600 ncu --metrics $M --clock-control none --csv \
    --log-file $O/${T}_launch_cfg$1_$2.csv $C2 > /dev/null 2>&1; echo "launch list cfg$1 $2 rc=$?"
done
for op in adjoint synthesize; do
  timeout 600 ncu --metrics $M --clock-control none --csv --log-file $O/${T}_launch_edag_$op.csv \
    python tools/bcop.py symmetric_edag $op > /dev/null 2>&1; echo "launch list edag $op rc=$?"
done
timeout 300 python tools/bcbench.py > $O/${T}_bcbench.txt 2>&1; echo "bcbench rc=$?"
for c in 4 5; do timeout 300 python tools/levelbench.py --cfg $c --ops adjoint,synthesize --reps 20; done > $O/${T}_levels.txt 2>&1
