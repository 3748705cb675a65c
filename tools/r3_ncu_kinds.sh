#!/bin/bash
# ncu --set full of the step-table kernel for HCPS[4,2] and RHD on 8 emulated ranks (C4's
# comparison plans; SURVEY §8(d) names CPS and HCPS[4,2]), then the 1-GPU suite and smoke on
# the final build (gpurun, 1 GPU).  -> gpurun_out/nk/
set -u
O=gpurun_out/nk
mkdir -p $O
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
step ncu_hcps42 timeout 900 bash -c "ncu --set full --clock-control none --import-source on -k regex:ar_exec_kernel -s 2 -c 1 -o $O/ncu_exec_hcps42_emulated8_bf16_256MiB $B --force hcps:4,2 > $O/ncu_hcps42.log 2>&1"
step ncu_rhd timeout 900 bash -c "ncu --set full --clock-control none --import-source on -k regex:ar_exec_kernel -s 2 -c 1 -o $O/ncu_exec_rhd_emulated8_bf16_256MiB $B --force rhd > $O/ncu_rhd.log 2>&1"
step bench_hcps42 timeout 600 bash -c "python bench.py --force hcps:4,2 --no-cpu-baseline --no-e2e > $O/bench_hcps42.json 2> $O/bench_hcps42.err"
step bench_rhd timeout 600 bash -c "python bench.py --force rhd --no-cpu-baseline --no-e2e > $O/bench_rhd.json 2> $O/bench_rhd.err"
step bench_ring timeout 600 bash -c "python bench.py --force ring --no-cpu-baseline --no-e2e > $O/bench_ring.json 2> $O/bench_ring.err"
step pytest_gpu timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_1gpu.log 2>&1
step smoke timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_1gpu.log 2>&1
echo done >> $O/steps.txt
