#!/bin/bash
# streaming ceilings of the dense product's data movement; B-gather L1 policy A/B on Reddit
O=gpurun_out; mkdir -p $O
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
timeout 600 python tools/stream_ceiling.py --out $O/stream_ceiling.jsonl > $O/stream_ceiling.log 2>&1
echo "exit $?" >> $O/stream_ceiling.log
for r in 1 2 3; do
  for na in 0 1; do
    PSPMM_B_NA=$na timeout 300 python tools/cfg_time.py --workloads reddit --iters 21 --tag na$na >> $O/na_ab.jsonl 2>> $O/na_ab.err
  done
done
