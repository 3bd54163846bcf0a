cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; grep -E "passed|failed|FAILED" gpurun_out/pytest_gpu.log | tail -8
timeout 900 python bench.py --no-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc $?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_c5.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['kernel_ms_per_step'], d['roofline']['frac'])"
for c in C3; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc $?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'], d['kernel_ms_per_step'])"
done
