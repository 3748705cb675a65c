#!/bin/bash
# C2 with the final executor (one-shot / LL128 / step-table paths), N = 4 and 2 (gpurun
# --gpus 4): our GenTree plan, GenTree incl. NVLS (path-aware pick), NVLS, NCCL default;
# an LL128 CTA-count probe at 2 CTAs per SM; the 1-GPU test suite on this build.
# -> gpurun_out/r2c/
set -u
O=gpurun_out/r2c
mkdir -p $O
P=29900
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
for n in 4 2; do
  step c2_n$n timeout 900 bash -c "$(declare -f T); P=$((P+10+n)); T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans 'gentree;gentree+nvls;nvls' --timing eager,graph > $O/c2_n${n}_f32.jsonl 2> $O/c2_n${n}_f32.err"
  step c2bf_n$n timeout 900 bash -c "$(declare -f T); P=$((P+20+n)); T --nproc-per-node $n tools/harness.py sweep --dtype bf16 --plans 'gentree' --timing graph > $O/c2_n${n}_bf16.jsonl 2> $O/c2_n${n}_bf16.err"
  step ll296_n$n timeout 600 bash -c "$(declare -f T); P=$((P+30+n)); AR_LL128_CTAS=296 AR_LL128_MAX_KB=32768 T --nproc-per-node $n tools/harness.py sweep --plans gentree --dtype f32 --timing graph --no-nccl --sizes 2097152 4194304 8388608 16777216 33554432 > $O/ll296_n$n.jsonl 2> $O/ll296_n$n.err"
done
step pytest_1gpu timeout 1500 bash -c "CUDA_VISIBLE_DEVICES=0 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_1gpu.log 2>&1"
step smoke timeout 300 bash -c "CUDA_VISIBLE_DEVICES=0 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1"
echo done >> $O/steps.txt
