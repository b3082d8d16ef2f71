#!/bin/bash
# usage: scripts/gpu_ncu_k.sh TAG KERNEL_REGEX [bench args...] -- one full ncu capture
tag=$1; k=$2; shift 2
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
  -f -o gpurun_out/${tag} python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e "$@" \
  > gpurun_out/${tag}.log 2>&1
echo "$tag rc=$?"
