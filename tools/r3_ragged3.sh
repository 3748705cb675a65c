#!/bin/bash
# LL128 RAGGED-templated build (gpurun --gpus 4): smoke, same-process tests on GPU 0, C2 at
# N = 4, 3, 2 (fp32; aligned sizes) and ragged sizes (power of two + 4 bytes).  -> gpurun_out/rg3/
set -u
O=gpurun_out/rg3
mkdir -p $O
P=31000
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step smoke timeout 300 bash -c "CUDA_VISIBLE_DEVICES=0 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1"
step pytest_sameproc timeout 1200 bash -c "CUDA_VISIBLE_DEVICES=0 python -m pytest tests/test_gpu_sameproc.py -v -p no:cacheprovider > $O/pytest_sameproc.log 2>&1"
R="524292 1048580 2097156 4194308 8388612 16777220 33554436"
for n in 4 3 2; do
  step c2_n$n timeout 900 bash -c "$(declare -f T); P=$((31010+n*10)); T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans gentree --timing graph --no-nccl > $O/c2_n${n}_f32.jsonl 2> $O/c2_n${n}_f32.err"
  step rag_n$n timeout 900 bash -c "$(declare -f T); P=$((31110+n*10)); T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans gentree --timing graph --no-nccl --sizes $R > $O/rag_n${n}_f32.jsonl 2> $O/rag_n${n}_f32.err"
done
echo done >> $O/steps.txt
