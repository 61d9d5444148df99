#!/bin/bash
# Copy one tools/profile_round.sh run (gpurun_out/<tag>_*) into the tracked profiles/r02_* evidence files.
# usage: bash tools/refresh_profiles.sh r02i
cd "$(dirname "$0")/.."
T=$1; O=gpurun_out; P=profiles
bash tools/ncu_report.sh $O/${T}_prof_*.ncu-rep > $P/r02_ncu_summary.txt 2>/dev/null
cp $O/${T}_bench.json $P/r02_bench_final.json
cp $O/${T}_bcbench.txt $P/r02_bcbench.txt
{ echo "# per-level chain timings (tools/levelbench.py): whole chain for J = 1..levels, CUDA-graph replay (warm, cold L2) and eager (cold)"; cat $O/${T}_levels.txt; } > $P/r02_levels.txt
cp $O/${T}_launches.csv $P/r02_launches_bench.csv
python tools/launch_summary.py $O/${T}_launches.csv 11 > $P/r02_launches_bench_summary.txt
{ echo "# cfg5 grad step (4 x 4096^2 CDF 9/7 sym 5 levels + 15-tap R), one call, ncu launch list (serialised, cold): kernel, us, DRAM MB"; python tools/ncu_last.py $O/${T}_launch_cfg5_grad.csv 11; } > $P/r02_launches_cfg5_grad.txt
{ echo "# cfg4 W* chain (4096^2 db8 zero, 6 levels), one call, ncu launch list (serialised, cold): kernel, us, DRAM MB"; python tools/ncu_last.py $O/${T}_launch_cfg4_adjoint.csv 6; } > $P/r02_launches_cfg4_adjoint.txt
{ echo "# paper-literal symmetric_edag at the cfg3 shape (8 x 2048^2 CDF 9/7, 5 levels): W* chain then W chain (split synthesis + border fold), one call each, ncu launch list"; python tools/ncu_last.py $O/${T}_launch_edag_adjoint.csv 5; python tools/ncu_last.py $O/${T}_launch_edag_synthesize.csv 10; } > $P/r02_launches_edag.txt
python - <<'PY'
import json, re
s = open('profiles/r02_ncu_summary.txt').read()
blk = s[s.index('prof_blur_residual'):]
rd = float(re.search(r'dram__bytes_read.sum\s+Mbyte\s+([\d.]+)', blk).group(1))
wr = float(re.search(r'dram__bytes_write.sum\s+Mbyte\s+([\d.]+)', blk).group(1))
tot = sum(float(m.group(1)) for m in (re.search(r'us\s+([\d.]+) MB', l) for l in open('profiles/r02_launches_cfg4_adjoint.txt')) if m)
d = {"_source": "r02 final: ncu --set full of k_blur_ring<7,1> (profiles/r02_ncu_summary.txt) and the ncu launch list of one cfg4 W* chain (profiles/r02_launches_cfg4_adjoint.txt): dram__bytes_read.sum + dram__bytes_write.sum, bytes per launch / per chain",
     "blur_residual_adjoint": (rd + wr) * 1e6, "wstar_cfg4_chain": tot * 1e6}
json.dump(d, open('profiles/traffic.json', 'w'), indent=1)
print(d)
PY
