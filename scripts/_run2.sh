cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_conv_tc.py tests/test_gpu_ops.py -q -m gpu -p no:cacheprovider > gpurun_out/pt_conv.log 2>&1; echo "pytest rc $?"; grep -E "assert|Error|FAILED|passed|failed" gpurun_out/pt_conv.log | head -30
