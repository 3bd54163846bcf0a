#!/bin/bash
# ncu --set full on full-stage (256x256) launches of the main kernels of a C2 bench step (1 GPU).
# Launch indices: per outer iteration 1 gram, 5 scatter, 5 update, 10 conv; stage 3 (full) starts at iteration 50.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/b1.json 2>&1 || { echo "plain run failed"; exit 1; }
prof() { ncu --set full --clock-control none --import-source on -k "regex:$1" -s $2 -c $3 -o gpurun_out/prof_$4 $CMD > gpurun_out/ncu_$4.log 2>&1; echo "ncu $4 rc $?"; }
prof gram_tc_kernel 70 1 gram
prof conv_coil_kernel 1600 2 conv
prof scatter_coil_kernel 800 1 scatter
prof update_kernel 800 1 update
prof "hetrd|householder_kernel" 340 2 nullspace
