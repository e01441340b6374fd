#!/bin/bash
# round 2, call AA: decider supplement of small hub-heavy graphs (Cora-like), 21 launches per point
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 1800 python tools/sweep.py --corpus 12 --corpus-seed 779 --corpus-n 1500,9000 --corpus-prefix t \
  --corpus-kinds chung_lu,powerlaw --corpus-d 2,12 --iters 21 --modes 0,3 --orders 0,1 \
  --out $O/sweep_tiny_r02.json > $O/sweep_tiny.log 2>&1
echo "exit $?" >> $O/sweep_tiny.log
