#!/bin/bash
# ring-only dense product: GNN tests, forms A/B with the copy ceiling
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gnn.py -q -x > $O/pytest_gnn.log 2>&1
echo "pytest exit $?" >> $O/pytest_gnn.log
timeout 900 python tools/gemm_forms.py --out $O/gemm_forms.jsonl > $O/gemm_forms.log 2>&1
echo "forms exit $?" >> $O/gemm_forms.log
