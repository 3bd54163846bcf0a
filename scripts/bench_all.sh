#!/bin/bash
# All bench configurations on one GPU (driver-style lines), outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "C5 rc=$?"
for c in C1 C2 C4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "C3 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_C5.json 2> gpurun_out/bench_ref_C5.err; echo "ref rc=$?"
