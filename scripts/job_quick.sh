cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gram_lag.py tests/test_gpu_fullsize_properties.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
for c in C5 C4; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc $?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
print(round(d['value'],2), round(d['ms_per_step'],2), round(d['e2e']['value'],2), {k:round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gram.csv python scripts/gram_lag_profile.py C5 lag 2 > gpurun_out/gram_lag_profile.txt 2>&1; python scripts/summarize_launches.py gpurun_out/launches_gram.csv gpurun_out/launches_gram.md > /dev/null 2>&1; head -16 gpurun_out/launches_gram.md
