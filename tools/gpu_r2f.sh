#!/bin/bash
# round 2, call F: mode-5 v4 (even-padded pair runs) parity, A/B, ncu x2; gather ceilings
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_block.py -q -x > $O/pytest_block.log 2>&1
echo "pytest exit $?" >> $O/pytest_block.log
timeout 1200 python tools/block_ab.py --workloads proteins,proteins_clustered --out $O/block_ab.jsonl > $O/block_ab.log 2>&1
echo "block_ab exit $?" >> $O/block_ab.log
for RW in 8 16; do
PSPMM_BLOCK_RW=$RW timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_block -s 1 -c 1 \
  -o /tmp/prof_block_$RW -f python tools/run_kernel.py --workload proteins --iters 2 --V 1 --S 0 --mode 5 > $O/ncu_block_$RW.log 2>&1
cp /tmp/prof_block_$RW.ncu-rep $O/ 2>/dev/null
done
timeout 1200 python tools/gather_ceiling.py --out $O/gather_ceiling_r02.json > $O/gather_ceiling.log 2>&1
echo "gather exit $?" >> $O/gather_ceiling.log
