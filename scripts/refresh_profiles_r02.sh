#!/bin/bash
# Round-2 measurement artefacts in one gpurun call (1 GPU), headline config C5:
#   the default bench line, the ncu launch list of the same workload (one
#   warm-up + one timed + one profiled step), ncu --set full captures of the
#   main kernels (+ summary json/md), per-config supplementary lines.
# usage: scripts/refresh_profiles_r02.sh TAG   (outputs in gpurun_out/, copied to profiles/)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
T=${1:-r02}
timeout 1200 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err || { echo "bench failed"; tail gpurun_out/bench_$T.err; exit 1; }
tail -c 300 gpurun_out/bench_$T.json; echo
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
   --log-file gpurun_out/launches_$T.csv $CMD > gpurun_out/ncu_launches_$T.log 2>&1
echo "launch list rc $?"
python scripts/summarize_launches.py gpurun_out/launches_$T.csv gpurun_out/launches_$T.md > /dev/null 2>&1
prof() { timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s $2 -c $3 -o gpurun_out/prof_$4_$T -f $CMD > gpurun_out/ncu_$4_$T.log 2>&1; echo "ncu $4 rc $?"; }
prof "lagtc_core|lag_edge2" 2 2 gram
prof "conv_tri_kernel|conv_tc_kernel" 15 3 conv
prof "split_t_kernel|split_kernel|amax_kernel" 30 2 split
prof update_kernel 5 1 update
python scripts/ncu_summary.py gpurun_out/prof_gram_$T.ncu-rep gpurun_out/prof_conv_$T.ncu-rep gpurun_out/prof_split_$T.ncu-rep gpurun_out/prof_update_$T.ncu-rep \
    -o gpurun_out/ncu_full_summary_$T.md --json gpurun_out/ncu_full_$T.json > /dev/null 2>&1
echo "summary rc $?"
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_${c}_$T.json 2> gpurun_out/bench_${c}_$T.err
  echo "$c rc $?"
done
timeout 600 python scripts/shard_bench.py C5full C5 C3 --iters 2 > gpurun_out/shard_$T.jsonl 2>&1
ls gpurun_out/ | grep $T
