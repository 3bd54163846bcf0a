#!/bin/bash
# source-level stall sampling of one conv_tc launch of the C5 shard workload (1 GPU)
# usage: scripts/ncu_conv_src.sh regex tag [skip]
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k "regex:$1" -s ${3:-3} -c 1 \
    -o gpurun_out/prof_$2 -f python scripts/shard_bench.py C5 --iters 0 > gpurun_out/ncu_$2.log 2>&1; echo "rc $?"
