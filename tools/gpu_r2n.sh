#!/bin/bash
# round 2, call N: large-graph decider supplement (candidate labels only, 21 launches), band tests
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_band.py -q -x > $O/pytest_band.log 2>&1
echo "pytest exit $?" >> $O/pytest_band.log
timeout 600 python tools/mc_probe.py > $O/mc_probe.log 2>&1
echo "mc_probe exit $?" >> $O/mc_probe.log
timeout 2400 python tools/sweep.py --corpus 8 --corpus-seed 778 --corpus-n 800000,3000000 --corpus-prefix L \
  --iters 21 --modes 0,3 --orders 0,1 --candidates profiles/r01/sweeps/sweep_corpus_*.json profiles/r02/sweeps/sweep_small_r02.json \
  --out $O/sweep_large_r02.json > $O/sweep_large.log 2>&1
echo "large exit $?" >> $O/sweep_large.log
