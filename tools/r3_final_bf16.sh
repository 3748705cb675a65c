#!/bin/bash
# Final build after the bf16 pack change (gpurun --gpus 4): multi-GPU parity, bench N = 4/3/2 bf16,
# C2 bf16 sweeps N = 4/2, the 1-GPU suite on GPU 0.  -> gpurun_out/fb/
set -u
O=gpurun_out/fb
mkdir -p $O
P=31600
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_multi timeout 2700 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider > $O/pytest_multi.log 2>&1
for n in 4 3 2; do
  step bench_n${n}_bf16 timeout 600 bash -c "$(declare -f T); P=$((31610+n*10)); T --nproc-per-node $n bench.py --gpus $n > $O/bench_n${n}_bf16.json 2> $O/bench_n${n}_bf16.err"
done
for n in 4 2; do
  step c2bf_n$n timeout 900 bash -c "$(declare -f T); P=$((31710+n)); T --nproc-per-node $n tools/harness.py sweep --dtype bf16 --plans 'gentree' --timing graph > $O/c2_n${n}_bf16.jsonl 2> $O/c2_n${n}_bf16.err"
done
step bench_n1_bf16 timeout 600 bash -c "CUDA_VISIBLE_DEVICES=0 python bench.py > $O/bench_n1_bf16.json 2> $O/bench_n1_bf16.err"
echo done >> $O/steps.txt
