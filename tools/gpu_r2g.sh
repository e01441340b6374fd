#!/bin/bash
# round 2, call G: mode-5 warp-count instances: parity, A/B, ncu of 8x23
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_block.py -q -x > $O/pytest_block.log 2>&1
echo "pytest exit $?" >> $O/pytest_block.log
timeout 1200 python tools/block_ab.py --workloads proteins --out $O/block_ab.jsonl > $O/block_ab.log 2>&1
echo "block_ab exit $?" >> $O/block_ab.log
PSPMM_BLOCK_NW=23 timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_block -s 1 -c 1 \
  -o /tmp/prof_block_23 -f python tools/run_kernel.py --workload proteins --iters 2 --V 1 --S 0 --mode 5 > $O/ncu_block_23.log 2>&1
cp /tmp/prof_block_23.ncu-rep $O/ 2>/dev/null
