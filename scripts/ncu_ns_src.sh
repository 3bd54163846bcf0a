#!/bin/bash
# full ncu capture (source-level stall sampling at the finest interval) of the
# named nullspace kernels (1 GPU).  usage: scripts/ncu_ns_src.sh 'regex' tag [count]
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python scripts/nullspace_bench.py 3 || exit 1
ncu --set full --import-source on --clock-control none --warp-sampling-interval 0 -k "regex:$1" -c ${3:-1} \
    -o gpurun_out/prof_$2 -f python scripts/nullspace_bench.py 2 > gpurun_out/ncu_$2.log 2>&1
tail -2 gpurun_out/ncu_$2.log
