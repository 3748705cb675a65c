#!/bin/bash
# Emulated validation sweep in bf16 on the final build (gpurun, 1 GPU): 8 ranks, every kind,
# 1 MiB - 1 GiB, graph timing.  -> gpurun_out/eb/
set -u
O=gpurun_out/eb
mkdir -p $O
timeout 1500 python tools/harness.py emu-sweep --ranks 8 --dtype bf16 --timing graph --sizes 1048576 2097152 4194304 8388608 16777216 33554432 67108864 134217728 268435456 536870912 1073741824 > $O/val_emu8_bf16.jsonl 2> $O/val_emu8_bf16.err
echo "rc=$?" > $O/done.txt
