#!/bin/bash
# One gpurun call: GPU tests, smoke, a short bench, and the ncu launch list.
# Usage (from the repo root on the GPU box): bash tools/gpu_check.sh [pytest-args]
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | grep "Model name" >> gpurun_out/nproc.txt
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
timeout 1500 python -m pytest tests -m gpu -q --maxfail=25 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
