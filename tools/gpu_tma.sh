#!/bin/bash
# TMA gather experiments: microbenchmark, mode-2 parity, mode 0 vs 2 sweep.
set -u
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/mb tools/microbench_gather.cu > $O/mb_build.log 2>&1
timeout 300 /tmp/mb 232965 64 114615892 > $O/mb_reddit.log 2>&1
timeout 300 /tmp/mb 2449029 128 123718280 > $O/mb_products.log 2>&1
timeout 300 /tmp/mb 132534 256 79122504 > $O/mb_proteins.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spmm.py -q -k "tma" > $O/pytest_tma.log 2>&1
echo "exit $?" >> $O/pytest_tma.log
timeout 1200 python tools/sweep.py --workloads roadnet,reddit,proteins,products --VS 10,11 \
    --Ws 2,4,8 --iters 5 --modes 0,2 --out $O/sweep_modes.json > $O/sweep_modes.log 2>&1
