cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > gpurun_out/b1.json 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k "regex:gram_tc_kernel" -s 70 -c 1 -o gpurun_out/prof_gram2 $CMD > gpurun_out/ncu_gram2.log 2>&1; echo "rc $?"; ls -la gpurun_out/prof_gram2.ncu-rep
