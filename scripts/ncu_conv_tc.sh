#!/bin/bash
# Source-level ncu capture of conv_tc_kernel launches from scripts/conv_tc_bench.py (1 GPU).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python scripts/conv_tc_bench.py > gpurun_out/conv_tc_bench.json 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:conv_tc_kernel" -s 2 -c 1 \
    -o gpurun_out/prof_convtc_full python scripts/conv_tc_bench.py > gpurun_out/ncu_convtc.log 2>&1
echo "ncu rc $?"
