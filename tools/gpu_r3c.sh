#!/bin/bash
# dense product vs a plain device copy of the same bytes
O=gpurun_out; mkdir -p $O
timeout 600 python tools/gemm_forms.py --shapes 64x64,128x128 --variants direct,ring --out $O/gemm_copy.jsonl > $O/gemm_copy.log 2>&1
echo "exit $?" >> $O/gemm_copy.log
