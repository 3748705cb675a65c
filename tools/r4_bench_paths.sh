#!/bin/bash
# bench N=1 with the path-aware emulated GenModel (gpurun, 1 GPU): default (CPS on the flat
# kernel) and forced multi-step plans (step-table row).  -> gpurun_out/r4b/
set -u
O=gpurun_out/r4b
mkdir -p $O
timeout 600 python bench.py --no-e2e --no-cpu-baseline > $O/bench_n1_bf16.json 2> $O/bench_n1_bf16.err; echo "default rc=$?" >> $O/done.txt
for k in ring rhd rb "hcps:4,2"; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --force "$k" > "$O/bench_n1_bf16_$k.json" 2> "$O/bench_n1_bf16_$k.err"; echo "$k rc=$?" >> $O/done.txt
done
echo done >> $O/done.txt
