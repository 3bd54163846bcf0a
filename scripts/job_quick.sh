cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ops.py tests/test_gpu_reference_e2e.py tests/test_gpu_solver.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -5 gpurun_out/pytest_gpu.log
for c in C4 C3 C5; do
timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc $?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1])
print(round(d['value'],2), round(d['ms_per_step'],2), round(d['e2e']['value'],2), {k:round(v,2) for k,v in d['kernel_ms_per_step'].items()})"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 1500 --csv --log-file gpurun_out/launches_C4.csv python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches_C4.log 2>&1; echo "launches rc $?"
python scripts/summarize_launches.py gpurun_out/launches_C4.csv gpurun_out/launches_C4.md > /dev/null 2>&1; grep -E "hetrd|chol_cl" gpurun_out/launches_C4.md
