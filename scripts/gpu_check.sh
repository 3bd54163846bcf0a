#!/bin/bash
# one gpurun call: GPU tests, smoke, TF32 peak
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
if [ "$1" == "peak" ]; then timeout 300 python scripts/measure_tf32_peak.py > gpurun_out/tf32.log 2>&1; fi
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log
