#!/bin/bash
# warm per-kernel times of the nullspace pipeline (1 GPU)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python scripts/nullspace_bench.py 30 || exit 1
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -c 200 --csv \
    --log-file gpurun_out/ns_launches.csv python scripts/nullspace_bench.py 10 > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/ns_launches.csv 2>&1 | head -30
