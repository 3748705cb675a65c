#!/bin/bash
# LL128 for any count (gpurun --gpus 4): same-process tests on GPU 0, multi-GPU parity, C2 at
# N = 4, 3, 2 (fp32, GenTree; NCCL default alongside).  -> gpurun_out/rg/
set -u
O=gpurun_out/rg
mkdir -p $O
P=30800
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_sameproc timeout 1200 bash -c "CUDA_VISIBLE_DEVICES=0 python -m pytest tests/test_gpu_sameproc.py -v -p no:cacheprovider > $O/pytest_sameproc.log 2>&1"
step pytest_multi timeout 2400 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider -k "multi_process_bit_exact" > $O/pytest_multi.log 2>&1
for n in 4 3 2; do
  step c2_n$n timeout 900 bash -c "$(declare -f T); P=$((30810+n*10)); T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans gentree --timing graph > $O/c2_n${n}_f32.jsonl 2> $O/c2_n${n}_f32.err"
done
echo done >> $O/steps.txt
