#!/bin/bash
# A/B library variants on the big workloads (run on the GPU box).
# usage: bash tools/ab_variants.sh name1 name2 ...   ("main" = the default build)
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = main ]; then unset PSPMM_LIB; else export PSPMM_LIB=$PWD/paper_2605_15695_b200/variants/libpspmm_$v.so; fi
  timeout 900 python tools/sweep.py --workloads roadnet,reddit --VS 10,11,20 --Ws 2,4,8 --iters 5 --out gpurun_out/ab_${v}_small.json > gpurun_out/ab_${v}_small.log 2>&1
  timeout 900 python tools/sweep.py --workloads proteins,products --VS 11,10 --Ws 2,4 --iters 5 --out gpurun_out/ab_${v}_big.json > gpurun_out/ab_${v}_big.log 2>&1
done
