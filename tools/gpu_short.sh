#!/bin/bash
# (build the variant libraries first: python tools/variants.py shortreg=PSPMM_SHORT_RING=0 ringcg=PSPMM_SHORT_RING=1,PSPMM_SHORT_RING_CG=1; main is then the register form)
# Engine mode 3 A/B: the cp.async ring form (main, .ca), the ring with .cg
# (variant ringcg) and the register form (variant shortreg): roadNet sweep
# per library, plus one ncu capture of the ring form.
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
SHORT_VARIANTS="main ringcg shortreg" bash tools/gpu_round.sh short_ab
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ring -s 1 -c 1 \
    -o /tmp/prof_ring -f python tools/run_kernel.py --workload roadnet --iters 2 --V 1 --S 0 \
    --mode 3 --W 2 --F 2 --G 4 > $O/ncu_ring.log 2>&1
python tools/ncu_summary.py /tmp/prof_ring.ncu-rep --json $O/ncu_ring.json > /dev/null 2>&1
