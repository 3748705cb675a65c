#!/bin/bash
# e2e chunk-count probe (gpurun, 1 GPU): bench N=1 with AR_E2E_CHUNKS = 8, 16, 32, 64.
set -u
O=gpurun_out/e2e
mkdir -p $O
for c in 8 16 32 64; do
  AR_E2E_CHUNKS=$c timeout 300 python bench.py --no-cpu-baseline --steps 10 > $O/bench_c$c.json 2> $O/bench_c$c.err
done
echo done > $O/done.txt
