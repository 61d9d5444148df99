#!/bin/bash
# A/B (after the register-cap change): PDL kinds off, short-run thresholds -- graph replay of cfg5 grad, cfg4/cfg3 W*
cd "$(dirname "$0")/../.."
run() { echo "== $*"; env "$@" timeout 100 python tools/graphbench.py --cfg 5 --op grad --reps 40 | tail -1; env "$@" timeout 100 python tools/graphbench.py --cfg 4 --op adjoint --reps 40 | tail -1; env "$@" timeout 100 python tools/graphbench.py --cfg 3 --op adjoint --reps 40 | tail -1; }
run WL_X=0
run WL_NO_PDL=
run WL_NO_PDL=b
run WL_NO_PDL=A
run WL_NO_PDL=bAS
run WL_SHORT_MAX=0
run WL_SHORT_MAX=2
run WL_SHORT_MAX=4
