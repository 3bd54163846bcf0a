cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_conv_tc.py tests/test_gpu_ops.py -x -q -m gpu -p no:cacheprovider > gpurun_out/pt_conv.log 2>&1; echo "pytest rc $?"; tail -30 gpurun_out/pt_conv.log
rm -f gpurun_out/split.jsonl
for d in 0 32; do HICU_CONV_TC_DEBUG=$d timeout 300 python scripts/conv_tc_split2.py >> gpurun_out/split.jsonl 2>>gpurun_out/split.err; done
cat gpurun_out/split.jsonl; tail -3 gpurun_out/split.err
