#!/bin/bash
# Per-tile event timeline of ws_core16_kernel, CTA 0 (experiments build):
#   EXPS="0 166 678 1702" bash scripts/core_trace.sh
# bits: 2 no gathers, 4 no G GEMM, 32 no r D tile, 128 no TMEM loads,
#       512 no C GEMM, 1024 no COO copies.  The library in the snapshot must
# be an experiments build (make EXPERIMENTS=1).
mkdir -p gpurun_out
for e in ${EXPS:-0 166}; do
  FTKCU_WS_EXP=$e FTKCU_TRACE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e \
    --no-rmse-check --no-fp32-equiv > gpurun_out/trace_$e.json 2> gpurun_out/trace_$e.txt
  python -c "
import json; d=json.load(open('gpurun_out/trace_$e.json')); print('exp=$e', d['phases_ms'])"
  tail -65 gpurun_out/trace_$e.txt | awk 'NR>40 {print}' | head -3
done
