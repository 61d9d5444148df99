#!/bin/bash
# balanced vs banded runs: per-level chain timings (WL_BANDED set = banded)
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
run() {
timeout 300 python tools/levelbench.py --cfg 4 --ops adjoint,synthesize --reps 20
timeout 300 python tools/levelbench.py --cfg 5 --ops adjoint,synthesize --reps 20
timeout 300 python tools/opbench.py --cfg 5 --op grad
timeout 300 python tools/opbench.py --cfg 3 --op adjoint,synthesize,analyze
}
echo "== balanced"; run
echo "== banded"; export WL_BANDED=1; run
