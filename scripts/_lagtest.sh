cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram_lag.py tests/test_gpu_ops.py -q -p no:cacheprovider 2>&1 | grep -E "assert|Error|FAILED|passed|failed" | head -30
