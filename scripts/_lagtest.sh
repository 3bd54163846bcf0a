cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gram_lag.py -x -q -s -p no:cacheprovider -k "c5_shard" 2>&1 | grep -i "err"
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc $?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_c5.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kernel_ms_per_step'])"
tail -3 gpurun_out/bench_c5.err
