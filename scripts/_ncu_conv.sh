cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k "regex:conv_tc_kernel" -s 3 -c 1 -o gpurun_out/prof_conv_src -f python scripts/conv_tc_split2.py > gpurun_out/ncu_conv_src.log 2>&1; echo "rc $?"; tail -3 gpurun_out/ncu_conv_src.log
