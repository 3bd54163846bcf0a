cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for c in C4 C3 C2; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches_$c.log 2>&1; echo "rc $?"
python scripts/summarize_launches.py gpurun_out/launches_$c.csv gpurun_out/launches_$c.md > /dev/null 2>&1; head -22 gpurun_out/launches_$c.md
done
