#!/bin/bash
# one gpurun call: bench (plain) then the ncu launch list of the same command
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python bench.py --steps ${STEPS:-3} --warmup ${WARMUP:-3} > gpurun_out/bench.json 2> gpurun_out/bench.err
rc=$?
echo "bench exit $rc"
tail -c 3000 gpurun_out/bench.json
if [ $rc -eq 0 ] && [ "$NCU" == "1" ]; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
     --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu \
     > gpurun_out/ncu_bench.log 2>&1
  echo "ncu exit $?"
fi
