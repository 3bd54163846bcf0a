cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cur.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches_cur.log 2>&1; echo "rc $?"
python scripts/summarize_launches.py gpurun_out/launches_cur.csv gpurun_out/launches_cur.md > /dev/null 2>&1; head -40 gpurun_out/launches_cur.md
