#!/bin/bash
# round 2, call A: gather ceilings (workload streams, K-slices) + GPU suite
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
(nproc; lscpu | grep "Model name") > $O/host.txt 2>&1
timeout 1200 python tools/gather_ceiling.py --out $O/gather_ceiling_r02.json > $O/gather_ceiling.log 2>&1
echo "gather exit $?" >> $O/gather_ceiling.log
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
