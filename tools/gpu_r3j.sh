#!/bin/bash
# griddepcontrol.wait moved to the S = 1 write-back, float4 zeroing: parity + Reddit / Cora timing
O=gpurun_out; mkdir -p $O
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_fanout.py tests/test_gpu_full.py -q -x > $O/pytest_s1.log 2>&1
echo "pytest exit $?" >> $O/pytest_s1.log
timeout 600 python bench.py --headline-only --no-cusparse --steps 30 --warmup 5 > $O/bench_reddit.log 2>&1
timeout 600 python bench.py --workload cora --headline-only --no-cusparse --steps 30 --warmup 5 > $O/bench_cora.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
      --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --headline-only --no-cusparse > $O/bench_ncu.log 2>&1
