#!/bin/bash
# 8 ranks' communicators on one GPU (gpurun, 1 GPU): the same-process tests incl. N = 8
# (one-shot, LL128, flag path), then the whole GPU suite and smoke.  -> gpurun_out/n8/
set -u
O=gpurun_out/n8
mkdir -p $O
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step sameproc timeout 1500 python -m pytest tests/test_gpu_sameproc.py -v -p no:cacheprovider > $O/pytest_sameproc.log 2>&1
step pytest_gpu timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_1gpu.log 2>&1
step smoke timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_1gpu.log 2>&1
echo done >> $O/steps.txt
