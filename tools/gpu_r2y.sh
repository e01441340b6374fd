#!/bin/bash
# round 2, call Y: column-blocked tensor-core GEMM for large W
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gnn.py -q -x > $O/pytest_gnn.log 2>&1
echo "pytest exit $?" >> $O/pytest_gnn.log
timeout 900 python tools/gemm_ab.py --out $O/gemm_ab.jsonl > $O/gemm_ab.log 2>&1
echo "gemm_ab exit $?" >> $O/gemm_ab.log
