#!/bin/bash
# N > 1 bench flow rehearsed on one GPU (2 processes, gloo; not a measurement):
# Reddit with every exchange leg (auto: allgather, fanout, multicast), roadNet (auto: halo, allgather)
O=gpurun_out; mkdir -p $O
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
for w in reddit roadnet; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 \
      --dist-backend gloo --workload $w --no-cusparse > $O/rehearse_$w.log 2>&1
  echo "exit $?" >> $O/rehearse_$w.log
done
timeout 120 python bench.py --gpus 2 > $O/gpus2_guard.log 2>&1
echo "exit $?" >> $O/gpus2_guard.log
