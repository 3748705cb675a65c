#!/bin/bash
# Session re-entry check (gpurun, 1 GPU): the 1-GPU test suite, smoke and bench N=1 on the
# current build.  Outputs in gpurun_out/v1/.
set -u
O=gpurun_out/v1
mkdir -p $O
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_gpu timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_1gpu.log 2>&1
step smoke timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_1gpu.log 2>&1
step bench_bf16 timeout 600 bash -c "python bench.py > $O/bench_n1_bf16.json 2> $O/bench_n1_bf16.err"
echo done >> $O/steps.txt
