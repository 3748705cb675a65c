#!/bin/bash
# C2 with the re-tuned path cut-offs (LL128 from 768 KiB/(N-1) to 64 MiB/N), N = 4 and 2
# (gpurun --gpus 4): GenTree, GenTree incl. NVLS, NVLS and NCCL default (fp32), GenTree and
# NCCL default (bf16); multi-GPU parity; the 1-GPU test suite and smoke.  -> gpurun_out/r3c/
set -u
O=gpurun_out/r3c
mkdir -p $O
P=30200
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_multi timeout 2400 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider > $O/pytest_multi.log 2>&1
for n in 4 2; do
  step c2_n$n timeout 900 bash -c "$(declare -f T); P=$((P+10+n)); T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans 'gentree;gentree+nvls;nvls' --timing eager,graph > $O/c2_n${n}_f32.jsonl 2> $O/c2_n${n}_f32.err"
  step c2bf_n$n timeout 900 bash -c "$(declare -f T); P=$((P+20+n)); T --nproc-per-node $n tools/harness.py sweep --dtype bf16 --plans 'gentree' --timing graph > $O/c2_n${n}_bf16.jsonl 2> $O/c2_n${n}_bf16.err"
done
step pytest_1gpu timeout 1500 bash -c "CUDA_VISIBLE_DEVICES=0 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_1gpu.log 2>&1"
step smoke timeout 300 bash -c "CUDA_VISIBLE_DEVICES=0 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1"
echo done >> $O/steps.txt
