#!/bin/bash
# C2 at N = 3 on the final build (gpurun --gpus 4): fp32 GenTree / GenTree incl. NVLS / NVLS with
# NCCL default, NCCL Ring, bf16 GenTree with NCCL default.  -> gpurun_out/n3/
set -u
O=gpurun_out/n3
mkdir -p $O
P=31800
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step c2_n3 timeout 900 bash -c "$(declare -f T); P=31811; T --nproc-per-node 3 tools/harness.py sweep --dtype f32 --plans 'gentree;gentree+nvls;nvls' --timing eager,graph > $O/c2_n3_f32.jsonl 2> $O/c2_n3_f32.err"
step c2ring_n3 timeout 600 bash -c "$(declare -f T); P=31821; NCCL_ALGO=Ring T --nproc-per-node 3 tools/harness.py sweep --dtype f32 --plans none --timing eager,graph > $O/c2_n3_f32_ncclring.jsonl 2> $O/c2_n3_f32_ncclring.err"
step c2bf_n3 timeout 900 bash -c "$(declare -f T); P=31831; T --nproc-per-node 3 tools/harness.py sweep --dtype bf16 --plans 'gentree' --timing graph > $O/c2_n3_bf16.jsonl 2> $O/c2_n3_bf16.err"
echo done >> $O/steps.txt
