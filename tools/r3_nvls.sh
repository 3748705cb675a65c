#!/bin/bash
# Round-2 session-3 NVLS campaign (gpurun --gpus 4): dump the switch's bf16 results for the
# rounding analysis (N = 2, 3, 4), then sweep the NVLS kernel's vectors in flight per thread
# (AR_NVLS_U) x CTA count at N = 4 and 2, fp32 and bf16.  Outputs in gpurun_out/nv/.
set -u
O=gpurun_out/nv
mkdir -p $O
P=29800
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step sameproc_multilevel timeout 600 python -m pytest tests/test_gpu_sameproc.py -k multi_level -q -p no:cacheprovider > $O/pytest_sameproc_multilevel.log 2>&1
for n in 2 3 4; do
  step dump_n$n timeout 300 bash -c "$(declare -f T); P=$((P+n)); T --nproc-per-node $n tools/nvls_dump.py $O > $O/dump_n$n.log 2>&1"
done
S="16777216 268435456 1073741824"
for n in 4 2; do
  if [ $n = 4 ]; then US="4 8 16 2"; CS="16 32 64 8"; else US="4 8 16"; CS="16 32 64"; fi
  for u in $US; do
    for c in $CS; do
      step sw_n${n}_u${u}_c${c} timeout 300 bash -c "$(declare -f T); P=$((P+10+n*100+u*5+c)); AR_NVLS_U=$u AR_NVLS_CTAS=$c T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans nvls --no-nccl --timing graph --sizes $S > $O/sw_n${n}_u${u}_c${c}_f32.jsonl 2> $O/sw_n${n}_u${u}_c${c}.err"
    done
  done
done
echo done >> $O/steps.txt
