#!/bin/bash
# Ring K = 1 vs strata at P = 8, cells in mode-3 runs (experiments build;
# FTKCU_WS_EXP=64 drops the per-warp fence before a cell count, 16 the
# write-back, 2 the gathers).
make -C paper_2404_10087_b200 clean >/dev/null; make -j8 -C paper_2404_10087_b200 EXPERIMENTS=1 >/dev/null 2>&1
for e in 0 64 16 2 18; do
  FTKCU_WS_EXP=$e timeout 600 python scripts/dsgd_emulate.py --parts 8 --schedule strata --runs 2>/dev/null | grep parts | sed "s/^/exp=$e /"
  FTKCU_WS_EXP=$e timeout 600 python scripts/dsgd_emulate.py --parts 8 --schedule ring --tokens 1 --runs 2>/dev/null | grep parts | sed "s/^/exp=$e /"
done | python -c "
import json,sys
for l in sys.stdin:
    h, j = l.split('{',1); d=json.loads('{'+j); print(h, d['schedule'], d.get('tokens'), round(d['factor_ms'],3), round(d['core_ms'],3), round(d['epoch_ms'],3), '%.3g'%d['implied_job_nnz_per_s'])"
make -C paper_2404_10087_b200 clean >/dev/null; make -j8 -C paper_2404_10087_b200 >/dev/null 2>&1
