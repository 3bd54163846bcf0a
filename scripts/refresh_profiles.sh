#!/bin/bash
# One gpurun call that regenerates the round's measurement artefacts (1 GPU):
#   bench line, ncu launch list of the same command, ncu --set full captures of
#   full-stage launches of the main kernels (+ summary), shard/Gram supplementary benches.
# usage: scripts/refresh_profiles.sh TAG   (outputs under gpurun_out/, copied to profiles/ by hand)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
T=${1:-vX}
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err || { echo "bench failed"; exit 1; }
tail -c 400 gpurun_out/bench_$T.json
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
   --log-file gpurun_out/launches_$T.csv $CMD > gpurun_out/ncu_launches_$T.log 2>&1
echo "launch list rc $?"
python scripts/summarize_launches.py gpurun_out/launches_$T.csv > gpurun_out/launches_$T.md 2>&1
prof() { timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s $2 -c $3 -o gpurun_out/prof_$4_$T -f $CMD > gpurun_out/ncu_$4_$T.log 2>&1; echo "ncu $4 rc $?"; }
prof gram_tc_kernel 70 1 gram
prof conv_tc_kernel 1050 3 conv
prof update_kernel 350 1 update
prof "hetrd6|nsjl" 140 2 nullspace
python scripts/ncu_summary.py gpurun_out/prof_gram_$T.ncu-rep gpurun_out/prof_conv_$T.ncu-rep gpurun_out/prof_update_$T.ncu-rep \
    gpurun_out/prof_nullspace_$T.ncu-rep -o gpurun_out/ncu_full_summary_$T.md --json gpurun_out/ncu_full_$T.json > /dev/null 2>&1
echo "summary rc $?"
timeout 600 python scripts/shard_bench.py C3 C5 --iters 2 > gpurun_out/shard_$T.jsonl 2>&1
timeout 300 python scripts/gram_bench.py --big > gpurun_out/gram_$T.json 2>&1
timeout 300 python scripts/gram_accuracy.py > gpurun_out/gram_accuracy_$T.jsonl 2>&1
ls gpurun_out/ | grep $T
