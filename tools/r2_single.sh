#!/bin/bash
# Round-2 single-GPU campaign (gpurun, 1 GPU): tests, smoke, bench lines, ncu, emulated-rank
# GenModel data, CPU-oracle timing plan.  Outputs in gpurun_out/r2s/.
set -u
O=gpurun_out/r2s
mkdir -p $O
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_gpu timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_1gpu.log 2>&1
step smoke timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_1gpu.log 2>&1
step bench_bf16 timeout 600 bash -c "python bench.py > $O/bench_n1_bf16.json 2> $O/bench_n1_bf16.err"
step bench_f32 timeout 600 bash -c "python bench.py --dtype f32 > $O/bench_n1_f32.json 2> $O/bench_n1_f32.err"
step bench_ref timeout 600 bash -c "python bench.py --impl reference > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err"
B="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
step ncu_launches timeout 900 bash -c "ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_bench_n1.csv $B > $O/ncu_launches.log 2>&1"
step ncu_full timeout 1200 bash -c "ncu --set full --clock-control none --import-source on -k regex:ar_flat_kernel -s 2 -c 1 -o $O/ncu_flat_emulated8_bf16_256MiB $B > $O/ncu_full.log 2>&1"
step emu_cps timeout 900 bash -c "python tools/harness.py emu-cps --timing graph > $O/cps_emu.jsonl 2> $O/cps_emu.err"
step emu_val timeout 1200 bash -c "python tools/harness.py emu-sweep --ranks 8 --timing graph --sizes 1048576 2097152 4194304 8388608 16777216 33554432 67108864 134217728 268435456 536870912 1073741824 > $O/val_emu8.jsonl 2> $O/val_emu8.err"
step cpu_oracle timeout 1500 bash -c "python bench.py --cpu-timing-plan > $O/cpu_oracle_timing.jsonl 2> $O/cpu_oracle_timing.err"
echo done >> $O/steps.txt
