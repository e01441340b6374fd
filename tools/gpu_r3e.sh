#!/bin/bash
# after the mode-4 retirement: the GPU suite (sanitizer tests skip on this pool)
O=gpurun_out; mkdir -p $O
export PSPMM_GEN_CACHE=/tmp/pspmm_gen_cache
timeout 2400 python -m pytest tests -m gpu -q --maxfail=25 > $O/pytest_gpu.log 2>&1
echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke exit $?" >> $O/smoke.log
