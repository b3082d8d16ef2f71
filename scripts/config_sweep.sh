#!/bin/bash
# Bench line per BASELINE config (C2 headline, C3 Yahoo, C4 order 6, C5 rank sweep).
mkdir -p gpurun_out
tag=${1:-r01}
for a in "--config yahoo" "--config order6" "--rank 8" "--rank 16" "--rank 64" "--rank 128" "--config c1"; do
  timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 $a 2>>gpurun_out/sweep_$tag.err | tail -1 >> gpurun_out/sweep_$tag.jsonl
  echo "$a rc=$?"
done
