#!/bin/bash
# round 2, call M: mode 6 v2 (one-descriptor bulk staging), mode 5 every-lane release, sanitizers, multicast
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_band.py tests/test_gpu_block.py -q -x > $O/pytest_band.log 2>&1
echo "pytest exit $?" >> $O/pytest_band.log
timeout 900 python tools/band_ab.py --workloads roadnet --Ks 16,32,64,128 --out $O/band_ab.jsonl > $O/band_ab.log 2>&1
echo "band_ab exit $?" >> $O/band_ab.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm_band -s 1 -c 1 \
  -o /tmp/prof_band -f python tools/run_kernel.py --workload roadnet --iters 2 --V 1 --S 0 --mode 6 > $O/ncu_band.log 2>&1
cp /tmp/prof_band.ncu-rep $O/ 2>/dev/null
timeout 900 python tools/block_ab.py --workloads proteins --variants 8x23 --out $O/block_ab.jsonl > $O/block_ab.log 2>&1
echo "block_ab exit $?" >> $O/block_ab.log
timeout 1200 python -m pytest tests/test_gpu_sanitizer.py -q > $O/pytest_san.log 2>&1
echo "pytest exit $?" >> $O/pytest_san.log
timeout 600 python tools/mc_probe.py > $O/mc_probe.log 2>&1
echo "mc_probe exit $?" >> $O/mc_probe.log
