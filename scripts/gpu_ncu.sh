#!/bin/bash
# Full ncu captures of the two hot sweeps (one launch each, after warm-up).
tag=${1:-r01}; shift
mkdir -p gpurun_out
for k in ws_factor ws_core; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -f -o gpurun_out/${tag}_$k python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e "$@" \
    > gpurun_out/${tag}_$k.log 2>&1
  echo "$k rc=$?"
done
