cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for l in 4 8 16; do
HICU_C3_LANES=$l timeout 900 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c3_$l.json 2> gpurun_out/bench_c3_$l.err; echo "lanes $l rc $?"
python -c "
import json;d=json.loads(open('gpurun_out/bench_c3_$l.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e']['value'])"
done
