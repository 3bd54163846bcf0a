cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out; rm -f gpurun_out/split.jsonl
for d in 0; do HICU_CONV_TC_DEBUG=$d timeout 300 python scripts/conv_tc_split2.py >> gpurun_out/split.jsonl 2>>gpurun_out/split.err; done
cat gpurun_out/split.jsonl; tail -3 gpurun_out/split.err
