#!/bin/bash
# round 2, call T: GEMM prologue fix + A/B + ncu; N>1 bench flow rehearsed on one GPU (gloo)
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gnn.py -q -x > $O/pytest_gnn.log 2>&1
echo "pytest exit $?" >> $O/pytest_gnn.log
timeout 900 python tools/gemm_ab.py --out $O/gemm_ab.jsonl > $O/gemm_ab.log 2>&1
echo "gemm_ab exit $?" >> $O/gemm_ab.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 1 -c 1 \
  -o /tmp/prof_gemm -f python -c "
import torch,sys; sys.path.insert(0,'.')
from paper_2605_15695_b200 import api
X=torch.rand((232965,64),device='cuda'); W=torch.rand((64,64),device='cuda'); T=torch.empty((232965,64),device='cuda')
for _ in range(3): api.pspmm_dense_gemm(X,W,T)
torch.cuda.synchronize()" > $O/ncu_gemm.log 2>&1
cp /tmp/prof_gemm.ncu-rep $O/ 2>/dev/null
bash tools/gpu_round.sh rehearse
