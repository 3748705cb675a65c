#!/bin/bash
# Session-3 final multi-GPU evidence (gpurun --gpus 4): multi-GPU parity incl. N = 3, the
# path-choice test, bench lines at N = 4, 3, 2 (bf16 and fp32).  -> gpurun_out/r3f/
set -u
O=gpurun_out/r3f
mkdir -p $O
P=30600
T() { P=$((P+1)); python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port $P "$@"; }
step() { local name=$1; shift; local t0=$(date +%s); echo "== $name" >> $O/steps.txt; "$@"; echo "   rc=$? $(( $(date +%s) - t0 ))s" >> $O/steps.txt; }
step pytest_paths timeout 600 bash -c "CUDA_VISIBLE_DEVICES=0 python -m pytest tests/test_gpu_sameproc.py -k path_choice -v -p no:cacheprovider > $O/pytest_paths.log 2>&1"
step pytest_multi timeout 2700 python -m pytest tests/test_gpu_multi.py -v -p no:cacheprovider > $O/pytest_multi.log 2>&1
for n in 4 3 2; do
  for dt in bf16 f32; do
    step bench_n${n}_$dt timeout 600 bash -c "$(declare -f T); P=$((30610+n*10)); T --nproc-per-node $n bench.py --gpus $n --dtype $dt > $O/bench_n${n}_$dt.json 2> $O/bench_n${n}_$dt.err"
  done
done
echo done >> $O/steps.txt
