#!/bin/bash
# K = 32 diagnostic: the lattice on the held-out workloads (where does the forest's pick land?)
O=gpurun_out; mkdir -p $O
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
timeout 1500 python tools/sweep.py --workloads cora,reddit,proteins,products --Ks 32 --iters 5 \
    --Ws 2,4,8 --VS 10,11 --orders 0,1 --out $O/sweep_k32.json > $O/sweep_k32.log 2>&1
echo "exit $?" >> $O/sweep_k32.log
