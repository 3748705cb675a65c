#!/bin/bash
# LL128 two-shot path on real NVLink (gpurun --gpus 4): multi-process parity, then busbw vs
# size with the path on (CTA counts 32 / 64 / 148) and off, N = 4 and 2.  -> gpurun_out/r2ll/
set -u
O=gpurun_out/r2ll
mkdir -p $O
P=29800
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_mp timeout 1800 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider -k "multi_process_bit_exact or push_protocol" > $O/pytest_mp.log 2>&1
S="524288 1048576 2097152 4194304 8388608 16777216 33554432"
for n in 4 2; do
  step off_n$n timeout 600 bash -c "$(declare -f T); P=$((P+10+n)); AR_LL128_MAX_KB=0 T --nproc-per-node $n tools/harness.py sweep --plans gentree --dtype f32 --timing eager,graph --no-nccl --sizes $S > $O/off_n$n.jsonl 2> $O/off_n$n.err"
  for c in 32 64 148; do
    step on_n${n}_c$c timeout 600 bash -c "$(declare -f T); P=$((P+20+n+c)); AR_LL128_MAX_KB=32768 AR_LL128_CTAS=$c T --nproc-per-node $n tools/harness.py sweep --plans gentree --dtype f32 --timing eager,graph --no-nccl --sizes $S > $O/on_n${n}_c$c.jsonl 2> $O/on_n${n}_c$c.err"
  done
  step on_n${n}_bf16 timeout 600 bash -c "$(declare -f T); P=$((P+300+n)); AR_LL128_MAX_KB=32768 T --nproc-per-node $n tools/harness.py sweep --plans gentree --dtype bf16 --timing graph --sizes $S > $O/on_n${n}_bf16.jsonl 2> $O/on_n${n}_bf16.err"
done
echo done >> $O/steps.txt
