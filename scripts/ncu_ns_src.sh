#!/bin/bash
# full ncu capture (with source-level stall sampling) of one launch of each
# named nullspace kernel (1 GPU).  usage: scripts/ncu_ns_src.sh 'regex' tag
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python scripts/nullspace_bench.py 3 || exit 1
ncu --set full --import-source on --clock-control none -k "regex:$1" -c ${3:-3} \
    -o gpurun_out/prof_$2 -f python scripts/nullspace_bench.py 2 > gpurun_out/ncu_$2.log 2>&1
tail -3 gpurun_out/ncu_$2.log
