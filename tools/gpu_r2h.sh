#!/bin/bash
# round 2, call H: decider label recheck (top-8 labels x 21 launches, round-robin)
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 3300 python tools/sweep.py --recheck profiles/r01/sweeps/sweep_*.json --corpus 60 --top 8 \
  --iters 21 --out $O/recheck_r02.json > $O/recheck.log 2>&1
echo "recheck exit $?" >> $O/recheck.log
