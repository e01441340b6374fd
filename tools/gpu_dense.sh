#!/bin/bash
# Engine mode 1 (dense tiles on tcgen05): parity tests, then timing and one
# ncu capture of the tensor-core kernel on the clustered proteins workload.
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_dense.py -x -q > $O/dense_main.log 2>&1; echo "exit $?" >> $O/dense_main.log
if grep -q "exit 0" $O/dense_main.log; then
  timeout 900 python tools/dense_ab.py --workloads proteins_clustered --dens ${DENS:-0.03,0.1} > $O/dense_ab.jsonl 2> $O/dense_ab.err
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_tc -s 1 -c 1 \
      -o /tmp/prof_dense -f python tools/run_kernel.py --workload proteins_clustered --iters 2 \
      --V 1 --S 0 --F 4 --G 8 --W 2 --order 1 --dense 0.1 > $O/ncu_dense.log 2>&1
  python tools/ncu_summary.py /tmp/prof_dense.ncu-rep --json $O/ncu_dense.json > /dev/null 2>&1
  ncu -i /tmp/prof_dense.ncu-rep --page details --csv > $O/ncu_dense_details.csv 2>/dev/null
fi
