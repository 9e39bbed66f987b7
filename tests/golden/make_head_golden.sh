#!/bin/bash
# Generates tests/golden/cfg5_l6_head.json -- the reference itself (oracle/_ref,
# the unmodified reference sources) on the headline workload, 729^3, first two
# cycles -- on the GPU host (about 130 GB of RAM; ~15 min of tree build and
# ~15 min per sweep on one core).  Virtual memory is capped so an allocation
# failure ends the run instead of the host.  Usage (from this container):
#   gpurun --timeout 5400 -- bash tests/golden/make_head_golden.sh
# then copy gpurun_out/cfg5_l6_head.json into tests/golden/.
set -e
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
ulimit -v 185000000
python tests/golden/make_goldens.py cfg5_l6_head > gpurun_out/head_golden.log 2>&1 || true
free -g >> gpurun_out/head_golden.log; cp tests/golden/cfg5_l6_head.json gpurun_out/ 2>/dev/null || true
tail -30 gpurun_out/head_golden.log
