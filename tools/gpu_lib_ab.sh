#!/bin/bash
# A/B of library variants on the decided configs: main vs $VARIANTS, two
# (build each variant first, e.g. python tools/variants.py git:HEAD~1=prev)
# alternating rounds.  usage: VARIANTS="bnoalloc" bash tools/gpu_lib_ab.sh
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
for round in 1 2; do
  for v in main ${VARIANTS}; do
    if [ "$v" = main ]; then unset PSPMM_LIB; else export PSPMM_LIB=$PWD/paper_2605_15695_b200/variants/libpspmm_$v.so; fi
    timeout 900 python tools/cfg_time.py --workloads ${WORKLOADS:-reddit,proteins,products} --tag $v >> $O/lib_ab.jsonl 2>> $O/lib_ab.err
  done
done
unset PSPMM_LIB
