#!/bin/bash
# round 2, call Q: mode 6 v5 (interleaved rows), GEMM depth variants, full GPU suite, bench
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_band.py -q -x > $O/pytest_band.log 2>&1
echo "pytest exit $?" >> $O/pytest_band.log
timeout 900 python tools/band_ab.py --workloads roadnet --Ks 16,32,64,128 --out $O/band_ab.jsonl > $O/band_ab.log 2>&1
echo "band_ab exit $?" >> $O/band_ab.log
timeout 900 python tools/gemm_ab.py --out $O/gemm_ab.jsonl > $O/gemm_ab.log 2>&1
echo "gemm_ab exit $?" >> $O/gemm_ab.log
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 1200 python bench.py > $O/bench.log 2>&1
echo "bench exit $?" >> $O/bench.log
