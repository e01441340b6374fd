#!/bin/bash
# round 2, call Z: mode 6 with 128-row blocks at K <= 16
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_band.py -q -x > $O/pytest_band.log 2>&1
echo "pytest exit $?" >> $O/pytest_band.log
timeout 900 python tools/band_ab.py --workloads roadnet --Ks 16,32 --out $O/band_ab.jsonl > $O/band_ab.log 2>&1
echo "band_ab exit $?" >> $O/band_ab.log
