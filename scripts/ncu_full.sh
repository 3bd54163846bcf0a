#!/bin/bash
# ncu --set full on full-stage (256x256) launches of the main kernels of a C2 bench step (1 GPU).
# Per outer iteration: 1 gram, 5 x (conv_tc<0>, conv_tc<2> scatter, conv_tc<1> ELS), 5 updates;
# stage 3 (full) starts at iteration 50.  Nullspace kernels: one launch each per iteration.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/b1.json 2>&1 || { echo "plain run failed"; exit 1; }
prof() { ncu --set full --clock-control none --import-source on -k "regex:$1" -s $2 -c $3 -o gpurun_out/prof_$4 $CMD > gpurun_out/ncu_$4.log 2>&1; echo "ncu $4 rc $?"; }
prof gram_tc_kernel 70 1 gram
prof conv_tc_kernel 1050 3 conv
prof update_kernel 350 1 update
prof "hetrd6|householder2" 140 2 nullspace
