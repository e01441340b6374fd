#!/bin/bash
# One GPU session: tests, smoke, bench (+ launch list), ncu captures of the
# engine on every workload, and (optionally) the decider sweep.
# usage: bash tools/gpu_round.sh [tests] [bench] [ncu] [sweep] [corpus]
set -u
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out
mkdir -p $O
want() { for a in "${ARGS[@]}"; do [ "$a" = "$1" ] && return 0; done; return 1; }
ARGS=("$@")
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $O/gpu.txt 2>&1
(nproc; lscpu | grep "Model name") > $O/host.txt 2>&1

if want tests; then
  timeout 2400 python -m pytest tests -m gpu -q --maxfail=25 > $O/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> $O/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
  echo "smoke exit $?" >> $O/smoke.log
fi
if want bench; then
  timeout 1500 python bench.py > $O/bench.log 2>&1
  echo "bench exit $?" >> $O/bench.log
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --headline-only --no-cusparse \
      > $O/bench_ncu.log 2>&1
fi
if want ncu; then
  # full captures are summarised here (JSON) and only the headline report is
  # kept: gpurun_out/ must stay under 64 MiB or nothing comes back
  for w in reddit roadnet products proteins cora proteins_clustered; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmm -s 1 -c 1 \
        -o /tmp/prof_$w -f python tools/run_kernel.py --workload $w --iters 2 > $O/ncu_$w.log 2>&1
    python tools/ncu_summary.py /tmp/prof_$w.ncu-rep --json $O/ncu_$w.json > /dev/null 2>&1
    ncu -i /tmp/prof_$w.ncu-rep --page details --csv > $O/ncu_${w}_details.csv 2>/dev/null
  done
  cp /tmp/prof_reddit.ncu-rep $O/ 2>/dev/null
  # engine mode 1: the tcgen05 dense-tile kernel on the clustered proteins graph
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_tc -s 1 -c 1 \
      -o /tmp/prof_dense -f python tools/run_kernel.py --workload proteins_clustered --iters 2 \
      --dense 0.1 > $O/ncu_dense.log 2>&1
  python tools/ncu_summary.py /tmp/prof_dense.ncu-rep --json $O/ncu_dense.json > /dev/null 2>&1
  ncu -i /tmp/prof_dense.ncu-rep --page details --csv > $O/ncu_dense_details.csv 2>/dev/null
fi
if want sweep; then
  timeout 1800 python tools/sweep.py --workloads cora,roadnet,reddit,proteins,products --iters 5 \
      --modes 0,2 --Ws 2,4,8 --out $O/sweep_workloads.json > $O/sweep_workloads.log 2>&1
fi
if want corpus; then
  timeout 3000 python tools/sweep.py --corpus 60 --Ks 16,32,64,128,256 --iters 5 --Ws 2,4 --modes 0,2 \
      --out $O/sweep_corpus.json > $O/sweep_corpus.log 2>&1
fi
if want sweep3; then
  # engine mode 3 (V = 1, S = 0 only): merged into the records above by
  # (graph, K) when the decider is trained
  timeout 900 python tools/sweep.py --workloads cora,roadnet,reddit,proteins,products --iters 5 \
      --VS 10 --modes 3 --out $O/sweep_workloads_m3.json > $O/sweep_workloads_m3.log 2>&1
  timeout 1800 python tools/sweep.py --corpus 60 --Ks 16,32,64,128,256 --iters 5 --VS 10 \
      --modes 3 --out $O/sweep_corpus_m3.json > $O/sweep_corpus_m3.log 2>&1
fi
if want sweep_order; then
  # mode-0 points with the length-sorted unit order (order = 1); merged by (graph, K)
  timeout 1200 python tools/sweep.py --workloads cora,roadnet,reddit,proteins,products --iters 5 \
      --Ws 2,4,8 --orders 1 --out $O/sweep_workloads_o1.json > $O/sweep_workloads_o1.log 2>&1
  timeout 2400 python tools/sweep.py --corpus 60 --Ks 16,32,64,128,256 --iters 5 --Ws 2,4 \
      --orders 1 --out $O/sweep_corpus_o1.json > $O/sweep_corpus_o1.log 2>&1
fi
if want tests4; then
  timeout 1800 python -m pytest tests -m gpu -q -k "short or fanout or accumulate or cli or host" \
      --maxfail=10 > $O/pytest_gpu4.log 2>&1
  echo "pytest exit $?" >> $O/pytest_gpu4.log
fi
if want quickbench; then
  timeout 900 python bench.py --headline-only > $O/bench_quick.log 2>&1
  echo "bench exit $?" >> $O/bench_quick.log
fi
if want rehearse; then
  # the N > 1 bench flow on one GPU: 2 processes, gloo, every exchange
  for ex in fanout allgather halo; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
        --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 \
        --dist-backend gloo --exchange $ex --workload reddit > $O/rehearse_$ex.log 2>&1
    echo "exit $?" >> $O/rehearse_$ex.log
  done
fi
if want short_ab; then
  for v in ${SHORT_VARIANTS:-main}; do
    if [ "$v" = main ]; then unset PSPMM_LIB; else export PSPMM_LIB=$PWD/paper_2605_15695_b200/variants/libpspmm_$v.so; fi
    timeout 600 python tools/sweep.py --workloads roadnet --VS 10 --modes 3 --Ws 2,4,8 --iters 9 \
        --out $O/short_$v.json > $O/short_$v.log 2>&1
  done
  unset PSPMM_LIB
fi
if want diag; then
  for w in reddit products; do
    timeout 600 python tools/e2e_diag.py --workload $w > $O/e2e_diag_$w.json 2> $O/e2e_diag_$w.log
  done
fi
# never let gpurun_out/ exceed the 64 MiB merge limit
if [ "$(du -sm $O | cut -f1)" -gt 56 ]; then rm -f $O/*.ncu-rep; fi
echo done > $O/round_done.txt
