#!/bin/bash
# source-level stall sampling of one full-stage gram_tc_kernel launch inside the C2 bench (1 GPU)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/b1.json 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k "regex:gram_tc_kernel" -s 70 -c 1 \
    -o gpurun_out/prof_gram_src -f $CMD > gpurun_out/ncu_gram_src.log 2>&1; echo "rc $?"
