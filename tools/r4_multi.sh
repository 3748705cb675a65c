#!/bin/bash
# Session-4 multi-GPU run (gpurun --gpus 4) -> gpurun_out/r4m/: A6x validation sweep of every
# plan kind on the final build (fp32, graph timing, 2 MiB - 1 GiB, N = 2, 3, 4), bench N = 2 / 4
# bf16 and the reference arm under torchrun at N = 4.
set -u
O=gpurun_out/r4m
mkdir -p $O
P=31300
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
S="2097152 4194304 8388608 16777216 33554432 67108864 134217728 268435456 536870912 1073741824"
for n in 4 3 2; do
  step val_n$n timeout 900 bash -c "$(declare -f T); P=$((P+10*n)); T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans 'gentree;cps;ring;rhd;rb;hcps:2,2' --timing graph --no-nccl --sizes $S > $O/val_n${n}.jsonl 2> $O/val_n${n}.err"
done
for n in 4 2; do
  step bench_n${n}_bf16 timeout 600 bash -c "$(declare -f T); P=$((P+100+10*n)); T --nproc-per-node $n bench.py --gpus $n > $O/bench_n${n}_bf16.json 2> $O/bench_n${n}_bf16.err"
done
step bench_ref_n4 timeout 600 bash -c "$(declare -f T); P=$((P+200)); T --nproc-per-node 4 bench.py --impl reference --gpus 4 > $O/bench_ref_n4.json 2> $O/bench_ref_n4.err"
echo done >> $O/steps.txt
