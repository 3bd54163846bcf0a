cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:conv_tc_kernel<.int.2" -s 2 -c 1 -o gpurun_out/prof_scatter_src -f python scripts/conv_tc_split2.py > gpurun_out/ncu_scatter_src.log 2>&1; echo "rc $?"
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:conv_tc_kernel<.int.0" -s 2 -c 1 -o gpurun_out/prof_conv0_src -f python scripts/conv_tc_split2.py > gpurun_out/ncu_conv0_src.log 2>&1; echo "rc $?"
