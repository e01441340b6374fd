#!/bin/bash
# Round-end confirmation: GPU suite + smoke + bench + ncu, then the K sweep.
bash tools/gpu_round.sh tests bench ncu
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
timeout 1500 python tools/k_sweep.py > gpurun_out/k_sweep.jsonl 2> gpurun_out/k_sweep.err
