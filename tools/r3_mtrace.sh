#!/bin/bash
# Steady-state phase trace of the step-table kernel on the final build (gpurun --gpus 4).
set -u
O=gpurun_out/mt
mkdir -p $O
AR_LL_MAX_KB=0 AR_LL128_MAX_KB=0 timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 31901 --nproc-per-node 4 tools/harness.py mtrace --plans gentree --dtype f32 --steady 8 --sizes 65536 4194304 33554432 > $O/mtrace_n4.jsonl 2> $O/mtrace_n4.err
echo "rc=$?" > $O/done.txt
