#!/bin/bash
# LL128 batched-load version (gpurun --gpus 4) -> gpurun_out/r2lb/
set -u
O=gpurun_out/r2lb
mkdir -p $O
P=30100
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step sameproc bash -c "CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_sameproc.py -q -x -p no:cacheprovider > $O/sameproc.log 2>&1"
if grep -q "passed" $O/sameproc.log && ! grep -q "failed" $O/sameproc.log; then
  step mp timeout 1500 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider -k "multi_process_bit_exact" > $O/mp.log 2>&1
  S="1048576 2097152 4194304 8388608 16777216 33554432"
  for n in 4 2; do
    step on_n$n timeout 600 bash -c "$(declare -f T); P=$((P+10+n)); AR_LL128_MAX_KB=32768 T --nproc-per-node $n tools/harness.py sweep --plans gentree --dtype f32 --timing eager,graph --no-nccl --sizes $S > $O/on_n$n.jsonl 2> $O/on_n$n.err"
  done
fi
echo done >> $O/steps.txt
