#!/bin/bash
# ncu --set full (source-level) of one nullspace kernel: $1 = kernel regex, $2 = tag
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python scripts/nullspace_bench.py 5 || exit 1
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k "regex:$1" -s 3 -c 1 -o gpurun_out/prof_$2 \
    python scripts/nullspace_bench.py 5 > gpurun_out/ncu_$2.log 2>&1
echo "ncu rc $?"
