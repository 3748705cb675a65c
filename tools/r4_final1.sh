#!/bin/bash
# Session-4 (last of round 2) single-GPU confirmation of HEAD (gpurun, 1 GPU): the 1-GPU test
# suite, smoke, bench N=1 bf16/fp32 and the reference arm.  -> gpurun_out/r4/
set -u
O=gpurun_out/r4
mkdir -p $O
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_gpu timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_1gpu.log 2>&1
step smoke timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_1gpu.log 2>&1
step bench_bf16 timeout 600 bash -c "python bench.py > $O/bench_n1_bf16.json 2> $O/bench_n1_bf16.err"
step bench_f32 timeout 600 bash -c "python bench.py --dtype f32 > $O/bench_n1_f32.json 2> $O/bench_n1_f32.err"
step bench_ref timeout 600 bash -c "python bench.py --impl reference > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err"
echo done >> $O/steps.txt
