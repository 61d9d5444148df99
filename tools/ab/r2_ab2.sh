#!/bin/bash
# A/B of ab/*.so builds on graph-replayed operators: bash tools/r2_ab2.sh "cfg op;cfg op" lib...
cd "$(dirname "$0")/../.."
SPECS="$1"; shift
for L in paper_1707_02018_b200/libwl.so "$@"; do echo "== $L"; IFS=';'; for spec in $SPECS; do IFS=' '; set -- $spec; WL_LIB=$L timeout 120 python tools/graphbench.py --cfg $1 --op $2 --reps 30; done; done 2>&1
