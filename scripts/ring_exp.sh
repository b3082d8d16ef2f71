#!/bin/bash
# Ring vs strata per-rank cost at P = 8 (experiments build; FTKCU_WS_EXP=64
# drops the per-warp fence before a cell count, 16 the write-back).
make -C paper_2404_10087_b200 clean >/dev/null; make -j8 -C paper_2404_10087_b200 EXPERIMENTS=1 >/dev/null 2>&1
for cfg in netflix yahoo; do
  timeout 600 python scripts/dsgd_emulate.py --config $cfg --parts 8 --schedule strata 2>/dev/null | grep parts | sed "s/^/$cfg exp=0 /"
  for K in 1 2; do for e in 0 64 16; do
    FTKCU_WS_EXP=$e timeout 600 python scripts/dsgd_emulate.py --config $cfg --parts 8 --schedule ring --tokens $K 2>/dev/null | grep parts | sed "s/^/$cfg exp=$e /"
  done; done
done | python -c "
import json,sys
for l in sys.stdin:
    h, j = l.split('{',1); d=json.loads('{'+j); print(h, d['schedule'], d.get('tokens'), round(d['factor_ms'],3), round(d['core_ms'],3), round(d['epoch_ms'],3), '%.3g'%d['implied_job_nnz_per_s'])"
make -C paper_2404_10087_b200 clean >/dev/null; make -j8 -C paper_2404_10087_b200 >/dev/null 2>&1
