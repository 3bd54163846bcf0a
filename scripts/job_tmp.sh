cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize_properties.py -q -s -p no:cacheprovider > gpurun_out/pytest_fullsize.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_fullsize.log
T=v6
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu"
prof() { timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s $2 -c $3 -o gpurun_out/prof_$4_$T -f $CMD > gpurun_out/ncu_$4_$T.log 2>&1; echo "ncu $4 rc $?"; }
prof "conv_tri_kernel|conv_tc_kernel" 15 3 conv
prof "split_t_kernel|split_kernel|amax_kernel" 30 2 split
