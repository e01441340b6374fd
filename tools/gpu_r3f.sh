#!/bin/bash
# W-in-TMEM dense product: tests, then forms A/B
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gnn.py -q -x > $O/pytest_gnn.log 2>&1
echo "pytest exit $?" >> $O/pytest_gnn.log
timeout 900 python tools/gemm_forms.py --shapes 128x128,64x128,128x64,64x256,128x256,64x64 --variants default,ring,wt128,ring_ob1,ring_xs4 --out $O/gemm_forms.jsonl > $O/gemm_forms.log 2>&1
echo "forms exit $?" >> $O/gemm_forms.log
