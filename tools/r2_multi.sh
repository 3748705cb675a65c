#!/bin/bash
# Round-2 multi-GPU measurement campaign (run through gpurun --gpus 4 from the repo root).
# Every step is bounded by its own timeout and logs into gpurun_out/r2m/; a failing step does
# not stop the others.  See profiles/round2/COMMANDS.md for what each output file feeds.
set -u
O=gpurun_out/r2m
mkdir -p $O
N=$(nvidia-smi -L | wc -l)
echo "gpus=$N" > $O/info.txt
nvidia-smi -q -d CLOCK | head -40 >> $O/info.txt
lscpu | head -20 >> $O/info.txt
P=29500
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }

# 1. multi-GPU parity (torchrun workers: 2 and 4 GPUs; NVLS incl. the NVLS GenTree plan kind)
step pytest_multi timeout 1500 python -m pytest tests/test_gpu_multi.py -q -x > $O/pytest_multi.log 2>&1

# 2. bench lines (N = 4 and 2, bf16 and fp32), NCCL default / Ring / NVLS-off inside
for n in 4 2; do
  for dt in bf16 f32; do
    step bench_n${n}_$dt timeout 600 bash -c "$(declare -f T); P=$((P+10*n)); T --nproc-per-node $n bench.py --gpus $n --dtype $dt > $O/bench_n${n}_$dt.json 2> $O/bench_n${n}_$dt.err"
  done
done

# 3. C2 sweep fp32 64 KiB - 1 GiB: our GenTree plan, GenTree incl. NVLS, NVLS; NCCL default
for n in 4 2; do
  step c2_n$n timeout 900 bash -c "$(declare -f T); P=$((P+100+n)); T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans 'gentree;gentree+nvls;nvls' --timing eager,graph > $O/c2_n${n}_f32.jsonl 2> $O/c2_n${n}_f32.err"
  step c2_ring_n$n timeout 600 bash -c "$(declare -f T); P=$((P+110+n)); NCCL_ALGO=Ring T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans none --timing eager,graph > $O/c2_n${n}_f32_ncclring.jsonl 2> $O/c2_n${n}_f32_ncclring.err"
  step c2_nvlsoff_n$n timeout 600 bash -c "$(declare -f T); P=$((P+120+n)); NCCL_NVLS_ENABLE=0 T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans none --timing eager,graph > $O/c2_n${n}_f32_ncclnvlsoff.jsonl 2> $O/c2_n${n}_f32_ncclnvlsoff.err"
done
# NCCL's algorithm choice per size (default env), logged once
step nccl_algo timeout 300 bash -c "$(declare -f T); P=$((P+130)); NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=TUNING NCCL_DEBUG_FILE=$O/nccl_tuning.%h.%p.log T --nproc-per-node 4 tools/harness.py nccl-algo --dtype f32 > $O/nccl_algo.jsonl 2> $O/nccl_algo.err"

# 4. GenModel: CPS fit rows (C3-iii) and the validation set, N = 2, 3, 4, 1 MiB - 1 GiB
for n in 2 3 4; do
  step cps_n$n timeout 600 bash -c "$(declare -f T); P=$((P+140+n)); T --nproc-per-node $n tools/harness.py cps --timing graph > $O/cps_n$n.jsonl 2> $O/cps_n$n.err"
  step val_n$n timeout 900 bash -c "$(declare -f T); P=$((P+150+n)); T --nproc-per-node $n tools/harness.py sweep --plans 'gentree;cps;ring;rhd;rb;hcps:2,2' --timing graph --no-nccl --sizes 1048576 2097152 4194304 8388608 16777216 33554432 67108864 134217728 268435456 536870912 1073741824 > $O/val_n$n.jsonl 2> $O/val_n$n.err"
done

# 5. push protocol (write-only) vs pull at 64 MiB - 1 GiB; entry fence A/B at small sizes
for n in 4 2; do
  step push_n$n timeout 600 bash -c "$(declare -f T); P=$((P+160+n)); AR_PUSH_MAX_MB=2048 T --nproc-per-node $n tools/harness.py sweep --plans gentree --dtype bf16 --timing graph --no-nccl --sizes 16777216 67108864 268435456 1073741824 > $O/push_n$n.jsonl 2> $O/push_n$n.err"
  step pull_n$n timeout 600 bash -c "$(declare -f T); P=$((P+170+n)); T --nproc-per-node $n tools/harness.py sweep --plans gentree --dtype bf16 --timing graph --no-nccl --sizes 16777216 67108864 268435456 1073741824 > $O/pull_n$n.jsonl 2> $O/pull_n$n.err"
done
for f in 0 1; do
  step fence$f timeout 600 bash -c "$(declare -f T); P=$((P+180+f)); AR_ENTRY_FENCE=$f AR_LL_MAX_KB=0 T --nproc-per-node 4 tools/harness.py sweep --plans gentree --dtype f32 --timing eager,graph --no-nccl --sizes 65536 1048576 4194304 16777216 > $O/fence${f}_n4.jsonl 2> $O/fence${f}_n4.err"
done

# 6. C3-ii fan-in probes (x-to-x / x-to-1, push / pull) and C3-iv (fan-in under NVLink AG traffic)
step p2p timeout 900 bash -c "$(declare -f T); P=$((P+190)); T --nproc-per-node 4 tools/harness.py p2p --dtype f32 > $O/p2p_n4.jsonl 2> $O/p2p_n4.err"
step fanin timeout 600 python tools/harness.py fanin > $O/fanin.jsonl 2> $O/fanin.err
step fanin_ag timeout 900 python tools/harness.py fanin-ag > $O/fanin_ag.jsonl 2> $O/fanin_ag.err
echo done >> $O/steps.txt
