#!/bin/bash
# bf16 pack via cvt.rn.bf16x2.f32 (gpurun, 1 GPU): the GPU suite, smoke, bench N=1 bf16 for CPS
# and the comparison plans.  -> gpurun_out/bp/
set -u
O=gpurun_out/bp
mkdir -p $O
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_gpu timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_1gpu.log 2>&1
step smoke timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_1gpu.log 2>&1
step bench_cps timeout 600 bash -c "python bench.py > $O/bench_cps_bf16.json 2> $O/bench_cps_bf16.err"
for k in ring rhd hcps:4,2 hcps:2,4; do
  step bench_$k timeout 300 bash -c "python bench.py --force $k --no-cpu-baseline --no-e2e > $O/bench_${k/:/}_bf16.json 2> $O/bench_${k/:/}_bf16.err"
done
echo done >> $O/steps.txt
