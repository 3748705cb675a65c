#!/bin/bash
# Path cut-offs with the LL128 path in place (gpurun --gpus 4): the GenTree plan (CPS) on its
# default paths, with the one-shot path off (LL128 from the smallest size), and with the LL128
# range raised to 64 MiB; fp32 and bf16, N = 4 and 2, graph timing.  Outputs in gpurun_out/cut/.
set -u
O=gpurun_out/cut
mkdir -p $O
P=30000
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
S="65536 131072 262144 393216 524288 786432 1048576 1572864 2097152 4194304 16777216 25165824 33554432 50331648 67108864"
for n in 4 2; do
  for dt in f32 bf16; do
    step def_n${n}_$dt timeout 600 bash -c "$(declare -f T); P=$((30010+n*10)); T --nproc-per-node $n tools/harness.py sweep --dtype $dt --plans gentree --no-nccl --timing graph --sizes $S > $O/def_n${n}_$dt.jsonl 2> $O/def_n${n}_$dt.err"
    step ll128all_n${n}_$dt timeout 600 bash -c "$(declare -f T); P=$((30110+n*10)); AR_LL_MAX_KB=0 AR_LL128_MAX_KB=65536 T --nproc-per-node $n tools/harness.py sweep --dtype $dt --plans gentree --no-nccl --timing graph --sizes $S > $O/ll128all_n${n}_$dt.jsonl 2> $O/ll128all_n${n}_$dt.err"
  done
done
echo done >> $O/steps.txt
