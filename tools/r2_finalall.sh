#!/bin/bash
# Final-build multi-GPU campaign (gpurun --gpus 4) -> gpurun_out/r2z/
set -u
O=gpurun_out/r2z
mkdir -p $O
P=30300
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_multi timeout 2400 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider > $O/pytest_multi.log 2>&1
for n in 4 2; do
  step bench_n${n}_bf16 timeout 600 bash -c "$(declare -f T); P=$((P+10*n)); T --nproc-per-node $n bench.py --gpus $n > $O/bench_n${n}_bf16.json 2> $O/bench_n${n}_bf16.err"
done
step bench_n4_f32 timeout 600 bash -c "$(declare -f T); P=$((P+50)); T --nproc-per-node 4 bench.py --gpus 4 --dtype f32 > $O/bench_n4_f32.json 2> $O/bench_n4_f32.err"
for n in 4 2; do
  step c2_n$n timeout 900 bash -c "$(declare -f T); P=$((P+100+n)); T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans 'gentree;gentree+nvls;nvls' --timing eager,graph > $O/c2_n${n}_f32.jsonl 2> $O/c2_n${n}_f32.err"
  step c2bf_n$n timeout 900 bash -c "$(declare -f T); P=$((P+200+n)); T --nproc-per-node $n tools/harness.py sweep --dtype bf16 --plans 'gentree' --timing graph > $O/c2_n${n}_bf16.jsonl 2> $O/c2_n${n}_bf16.err"
done
echo done >> $O/steps.txt
