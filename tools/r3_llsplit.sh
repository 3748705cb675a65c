#!/bin/bash
# LL128 + step-table split probe (gpurun --gpus 4).  Outputs in gpurun_out/llsplit/.
set -u
O=gpurun_out/llsplit
mkdir -p $O
P=30400
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
for n in 4 2; do
  step a_n$n timeout 600 bash -c "$(declare -f T); P=$((30410+n)); AR_LL128_MAX_KB=262144 T --nproc-per-node $n tools/ll128_exec_split.py > $O/a_n$n.jsonl 2> $O/a_n$n.err"
  step b_n$n timeout 600 bash -c "$(declare -f T); P=$((30420+n)); SPLIT_EXEC_CTAS=100 AR_LL128_MAX_KB=262144 T --nproc-per-node $n tools/ll128_exec_split.py > $O/b_n$n.jsonl 2> $O/b_n$n.err"
  step c_n$n timeout 600 bash -c "$(declare -f T); P=$((30430+n)); AR_LL128_CTAS=148 AR_LL128_MAX_KB=262144 T --nproc-per-node $n tools/ll128_exec_split.py > $O/c_n$n.jsonl 2> $O/c_n$n.err"
done
echo done >> $O/steps.txt
