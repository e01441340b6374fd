#!/bin/bash
# round 2 re-entry, call B: dense-product forms A/B (direct vs split rings),
# GNN tests on the new default, ncu of both forms with the source page
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gnn.py -q -x > $O/pytest_gnn.log 2>&1
echo "pytest exit $?" >> $O/pytest_gnn.log
timeout 900 python tools/gemm_forms.py --out $O/gemm_forms.jsonl > $O/gemm_forms.log 2>&1
echo "forms exit $?" >> $O/gemm_forms.log
for f in ring direct; do
  PSPMM_GEMM_FORM=$f timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 \
      -o /tmp/prof_gemm_$f -f python tools/gemm_run.py > $O/ncu_gemm_$f.log 2>&1
  python tools/ncu_summary.py /tmp/prof_gemm_$f.ncu-rep --json $O/ncu_gemm_$f.json > /dev/null 2>&1
  ncu -i /tmp/prof_gemm_$f.ncu-rep --page source --csv > $O/ncu_gemm_${f}_source.csv 2>/dev/null
  ncu -i /tmp/prof_gemm_$f.ncu-rep --page details --csv > $O/ncu_gemm_${f}_details.csv 2>/dev/null
done
