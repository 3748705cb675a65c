#!/bin/bash
# Emulated-rank fit data on the final build (gpurun, 1 GPU), bf16, graph timing: CPS rows at
# 2..8 ranks (the flat kernel's A6e row) and Ring rows at 3..7 ranks (the step-table kernel's
# row; 8 ranks held out).  -> gpurun_out/r4f/
set -u
O=gpurun_out/r4f
mkdir -p $O
S="1048576 2097152 4194304 8388608 16777216 33554432 67108864 134217728 268435456 536870912 1073741824"
timeout 900 python tools/harness.py emu-cps --max-ranks 8 --dtype bf16 --timing graph > $O/cps_emu_bf16.jsonl 2> $O/cps_emu_bf16.err
echo "cps rc=$?" >> $O/done.txt
for n in 3 4 5 6 7; do
  timeout 900 python tools/harness.py emu-sweep --ranks $n --plans ring --dtype bf16 --timing graph --sizes $S >> $O/ring_emu_bf16.jsonl 2>> $O/ring_emu_bf16.err
  echo "ring n=$n rc=$?" >> $O/done.txt
done
echo done >> $O/done.txt
