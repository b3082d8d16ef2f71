#!/bin/bash
# Core-sweep timing decomposition (FTKCU_WS_EXP bits, experiments build only):
#   2 = no gathers, 4 = no G GEMM, 32 = no r D tile
# for one and two epilogue groups (--core16 1 / 2).  Rebuilds the library with
# EXPERIMENTS=1 first and restores the production build at the end.
make -C paper_2404_10087_b200 clean >/dev/null; make -j8 -C paper_2404_10087_b200 EXPERIMENTS=1 >/dev/null 2>&1
for g in ${GROUPS_:-1 2}; do
  for e in ${EXPS:-0 2 4 32 6 38}; do
    FTKCU_WS_EXP=$e timeout 300 python bench.py --no-cpu --no-e2e --no-rmse-check --no-fp32-equiv \
      --core16 $g 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('core16=$g exp=$e', {k: round(v,3) for k,v in d['phases_ms'].items()}, 'roof', d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['peak']))"
  done
done
make -C paper_2404_10087_b200 clean >/dev/null; make -j8 -C paper_2404_10087_b200 >/dev/null 2>&1
