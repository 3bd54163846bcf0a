cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for c in C1 C2 C5; do timeout 600 python scripts/e2e_trace.py $c 2> gpurun_out/trace_$c.txt > /dev/null; echo "trace $c rc $?"; done
timeout 600 python scripts/e2e_profile.py C1 > gpurun_out/e2eprof_C1.txt 2>&1; echo "prof rc $?"
for c in C2 C4; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 3000 --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launches_$c.log 2>&1; echo "launches $c rc $?"
python scripts/summarize_launches.py gpurun_out/launches_$c.csv gpurun_out/launches_$c.md > /dev/null 2>&1
done
