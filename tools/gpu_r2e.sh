#!/bin/bash
# round 2, call E: mode-5 v3 (staged pairs) parity, A/B, ncu; full GPU suite; bench
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_block.py -q -x > $O/pytest_block.log 2>&1
echo "pytest exit $?" >> $O/pytest_block.log
timeout 1200 python tools/block_ab.py --workloads proteins,proteins_clustered,products --out $O/block_ab.jsonl > $O/block_ab.log 2>&1
echo "block_ab exit $?" >> $O/block_ab.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_block -s 1 -c 1 \
  -o /tmp/prof_block -f python tools/run_kernel.py --workload proteins --iters 2 --V 1 --S 0 --mode 5 > $O/ncu_block.log 2>&1
python tools/ncu_summary.py /tmp/prof_block.ncu-rep --json $O/ncu_block.json > /dev/null 2>&1
cp /tmp/prof_block.ncu-rep $O/ 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.log 2>&1
echo "bench exit $?" >> $O/bench.log
