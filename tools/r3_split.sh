#!/bin/bash
# NVLS + P2P side-by-side probe (gpurun --gpus 4).  Outputs in gpurun_out/split/.
set -u
O=gpurun_out/split
mkdir -p $O
P=29900
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step split_n4 timeout 600 bash -c "$(declare -f T); P=29911; T --nproc-per-node 4 tools/nvls_p2p_split.py > $O/split_n4.jsonl 2> $O/split_n4.err"
step split_n4_c8 timeout 600 bash -c "$(declare -f T); P=29921; AR_NVLS_CTAS=8 AR_NVLS_U=8 T --nproc-per-node 4 tools/nvls_p2p_split.py > $O/split_n4_c8.jsonl 2> $O/split_n4_c8.err"
step split_n2 timeout 600 bash -c "$(declare -f T); P=29931; T --nproc-per-node 2 tools/nvls_p2p_split.py > $O/split_n2.jsonl 2> $O/split_n2.err"
echo done >> $O/steps.txt
