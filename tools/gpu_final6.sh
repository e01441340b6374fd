#!/bin/bash
# Round-2 last run on the final code: GPU suite + smoke + bench + launch list + ncu of every workload, dense-product kernels, K sweep
bash tools/gpu_round.sh tests bench ncu
O=gpurun_out
for f in 64x64 128x128; do
  Ki=${f%x*}; Ko=${f#*x}
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 \
      -o /tmp/prof_gemm_$f -f python tools/gemm_run.py --Ki $Ki --Ko $Ko > $O/ncu_gemm_$f.log 2>&1
  python tools/ncu_summary.py /tmp/prof_gemm_$f.ncu-rep --json $O/ncu_gemm_$f.json > /dev/null 2>&1
done
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
timeout 1500 python tools/k_sweep.py > $O/k_sweep.jsonl 2> $O/k_sweep.err
rm -f $O/*.ncu-rep
echo done > $O/final_done.txt
