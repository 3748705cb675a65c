#!/bin/bash
# Session-3 final single-GPU evidence (gpurun, 1 GPU): the 1-GPU test suite, smoke, bench N=1
# bf16/fp32, the reference arm, the bench launch list, and an ncu --set full capture of the
# step-table kernel running the Ring plan on 8 emulated ranks (C4 comparison plan).
# -> gpurun_out/r3s/
set -u
O=gpurun_out/r3s
mkdir -p $O
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_gpu timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_1gpu.log 2>&1
step smoke timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_1gpu.log 2>&1
step bench_bf16 timeout 600 bash -c "python bench.py > $O/bench_n1_bf16.json 2> $O/bench_n1_bf16.err"
step bench_f32 timeout 600 bash -c "python bench.py --dtype f32 > $O/bench_n1_f32.json 2> $O/bench_n1_f32.err"
step bench_ref timeout 600 bash -c "python bench.py --impl reference > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err"
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
step ncu_launches timeout 900 bash -c "ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_bench_n1.csv $B > $O/ncu_launches.log 2>&1"
step ncu_ring timeout 1200 bash -c "ncu --set full --clock-control none --import-source on -k regex:ar_exec_kernel -s 2 -c 1 -o $O/ncu_exec_ring_emulated8_bf16_256MiB $B --force ring > $O/ncu_ring.log 2>&1"
echo done >> $O/steps.txt
