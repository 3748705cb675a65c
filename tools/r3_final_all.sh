#!/bin/bash
# Session-3 final evidence on the final build (gpurun --gpus 4): multi-GPU parity (N = 2, 3, 4;
# NVLS incl. AVG; ragged LL128), the 1-GPU suite + smoke on GPU 0, bench lines N = 1..4, the C2
# sweeps (fp32 GenTree / GenTree incl. NVLS / NVLS / NCCL default, bf16 GenTree / NCCL default),
# the reference arm and the bench launch list.  -> gpurun_out/fin/
set -u
O=gpurun_out/fin
mkdir -p $O
P=31200
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_1gpu timeout 1800 bash -c "CUDA_VISIBLE_DEVICES=0 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_1gpu.log 2>&1"
step smoke timeout 300 bash -c "CUDA_VISIBLE_DEVICES=0 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke_1gpu.log 2>&1"
step pytest_multi timeout 2700 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider > $O/pytest_multi.log 2>&1
step bench_n1_bf16 timeout 600 bash -c "CUDA_VISIBLE_DEVICES=0 python bench.py > $O/bench_n1_bf16.json 2> $O/bench_n1_bf16.err"
step bench_n1_f32 timeout 600 bash -c "CUDA_VISIBLE_DEVICES=0 python bench.py --dtype f32 > $O/bench_n1_f32.json 2> $O/bench_n1_f32.err"
step bench_ref timeout 600 bash -c "CUDA_VISIBLE_DEVICES=0 python bench.py --impl reference > $O/bench_ref_n1.json 2> $O/bench_ref_n1.err"
step ncu_launches timeout 900 bash -c "CUDA_VISIBLE_DEVICES=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ncu_launches_bench_n1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launches.log 2>&1"
for n in 4 3 2; do
  for dt in bf16 f32; do
    step bench_n${n}_$dt timeout 600 bash -c "$(declare -f T); P=$((31210+n*10)); T --nproc-per-node $n bench.py --gpus $n --dtype $dt > $O/bench_n${n}_$dt.json 2> $O/bench_n${n}_$dt.err"
  done
done
for n in 4 2; do
  step c2_n$n timeout 900 bash -c "$(declare -f T); P=$((31310+n)); T --nproc-per-node $n tools/harness.py sweep --dtype f32 --plans 'gentree;gentree+nvls;nvls' --timing eager,graph > $O/c2_n${n}_f32.jsonl 2> $O/c2_n${n}_f32.err"
  step c2bf_n$n timeout 900 bash -c "$(declare -f T); P=$((31320+n)); T --nproc-per-node $n tools/harness.py sweep --dtype bf16 --plans 'gentree' --timing graph > $O/c2_n${n}_bf16.jsonl 2> $O/c2_n${n}_bf16.err"
done
echo done >> $O/steps.txt
