#!/bin/bash
# Session-4 2-GPU check (gpurun --gpus 2) -> gpurun_out/r4n/: bench N=2 stdout is exactly one
# JSON line; the CPU-oracle timing plan on the GPU box's host (bench.py --cpu-timing-plan).
set -u
O=gpurun_out/r4n
mkdir -p $O
P=32300
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step bench_n2_f32 timeout 600 bash -c "$(declare -f T); T --nproc-per-node 2 bench.py --gpus 2 --dtype f32 > $O/bench_n2_f32.json 2> $O/bench_n2_f32.err"
step ref_n2 timeout 600 bash -c "$(declare -f T); P=$((P+5)); T --nproc-per-node 2 bench.py --impl reference --gpus 2 > $O/bench_ref_n2.json 2> $O/bench_ref_n2.err"
step cpu_timing timeout 1200 bash -c "python bench.py --cpu-timing-plan > $O/cpu_oracle_timing.jsonl 2> $O/cpu_oracle_timing.err"
echo done >> $O/steps.txt
