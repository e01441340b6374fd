#!/bin/bash
# round 2, call J: decider corpus supplements (small and large graphs), 21 launches per point
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 1200 python tools/sweep.py --corpus 18 --corpus-seed 777 --corpus-n 1000,20000 --corpus-prefix s \
  --iters 21 --modes 0,3 --orders 0,1 --out $O/sweep_small_r02.json > $O/sweep_small.log 2>&1
echo "small exit $?" >> $O/sweep_small.log
timeout 2400 python tools/sweep.py --corpus 8 --corpus-seed 778 --corpus-n 800000,3000000 --corpus-prefix L \
  --iters 21 --modes 0,3 --orders 0,1 --out $O/sweep_large_r02.json > $O/sweep_large.log 2>&1
echo "large exit $?" >> $O/sweep_large.log
