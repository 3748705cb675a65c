#!/bin/bash
# ar_flatsteps_kernel (gpurun, 1 GPU): emulated tests, then bench N=1 for the comparison plans
# with and without it (bf16 and fp32, 8 ranks x 256 MiB).  -> gpurun_out/fs/
set -u
O=gpurun_out/fs
mkdir -p $O
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_exec timeout 1500 python -m pytest tests/test_gpu_exec.py -q -p no:cacheprovider > $O/pytest_exec.log 2>&1
for k in ring rhd hcps:4,2 hcps:2,4 hcps:2,2,2; do
  for dt in bf16 f32; do
    for fs in 1 0; do
      step bench_${k}_${dt}_fs$fs timeout 300 bash -c "AR_FLATSTEPS=$fs python bench.py --force $k --dtype $dt --no-cpu-baseline --no-e2e > $O/bench_${k/:/}_${dt}_fs$fs.json 2> $O/bench_${k/:/}_${dt}_fs$fs.err"
    done
  done
done
echo done >> $O/steps.txt
