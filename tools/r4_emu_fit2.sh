#!/bin/bash
# Emulated multi-step fit rows (gpurun, 1 GPU), bf16, graph timing: RB, RHD and HCPS at 3..7
# ranks (8 ranks held out) for the step-table kernel's A6e row.  -> gpurun_out/r4g/
set -u
O=gpurun_out/r4g
mkdir -p $O
S="1048576 2097152 4194304 8388608 16777216 33554432 67108864 134217728 268435456 536870912 1073741824"
for n in 3 4 5 6 7; do
  timeout 900 python tools/harness.py emu-sweep --ranks $n --plans "rb;rhd;hcps:2,2;hcps:2,3;hcps:3,2" --dtype bf16 --timing graph --sizes $S >> $O/multistep_emu_bf16.jsonl 2>> $O/multistep_emu_bf16.err
  echo "n=$n rc=$?" >> $O/done.txt
done
echo done >> $O/done.txt
