#!/bin/bash
# Re-check after the extent fix (gpurun, 1 GPU): same-process tests, smoke.  -> gpurun_out/rg2/
set -u
O=gpurun_out/rg2
mkdir -p $O
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_sameproc timeout 1200 python -m pytest tests/test_gpu_sameproc.py -v -p no:cacheprovider > $O/pytest_sameproc.log 2>&1
step smoke timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo done >> $O/steps.txt
