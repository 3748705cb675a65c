#!/bin/bash
# Flakiness soak on the final build (gpurun, 1 GPU): pytest -m gpu x3, smoke x3.  -> gpurun_out/soak/
set -u
O=gpurun_out/soak
mkdir -p $O
for i in 1 2 3; do
  timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_$i.log 2>&1; echo "pytest $i rc=$?" >> $O/steps.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$i.log 2>&1; echo "smoke $i rc=$?" >> $O/steps.txt
done
echo done >> $O/steps.txt
