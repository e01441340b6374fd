#!/bin/bash
# round 2, call R: full GPU suite + smoke + bench + launch list + ncu of every workload + K sweep
bash tools/gpu_round.sh tests bench ncu
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
timeout 1500 python tools/k_sweep.py > gpurun_out/k_sweep.jsonl 2> gpurun_out/k_sweep.err
echo "ksweep exit $?" >> gpurun_out/k_sweep.err
