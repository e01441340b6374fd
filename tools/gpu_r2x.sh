#!/bin/bash
# round 2, call X: hub-prefix L2 persistence on degree-ordered products; CLI tests
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -k cli -q > $O/pytest_cli.log 2>&1
echo "pytest exit $?" >> $O/pytest_cli.log
timeout 1200 python tools/hub_l2_ab.py --workload products --out $O/hub_l2_ab.jsonl > $O/hub_l2_ab.log 2>&1
echo "exit $?" >> $O/hub_l2_ab.log
