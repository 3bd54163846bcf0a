cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram_lag.py tests/test_gpu_solver.py -x -q -p no:cacheprovider -k "lag or sharded or nccl" 2>&1 | tail -5
