#!/bin/bash
# dense product final defaults: tests + table
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gnn.py -q -x > $O/pytest_gnn.log 2>&1
echo "pytest exit $?" >> $O/pytest_gnn.log
timeout 900 python tools/gemm_forms.py --shapes 64x64,128x128,64x128,128x64,64x256,128x256 --variants default,ob2 --out $O/gemm_final.jsonl > $O/gemm_final.log 2>&1
echo "forms exit $?" >> $O/gemm_final.log
