#!/bin/bash
# Per-rank DSGD cost (one GPU emulating rank 0) for DESIGN.md §6: strata and
# ring (K = 1, 2), cells in mode-3 runs, P = 2, 4, 8; Yahoo at P = 8.
out=gpurun_out/dsgd_table.jsonl; rm -f $out
for P in 2 4 8; do
  timeout 300 python scripts/dsgd_emulate.py --parts $P --runs >> $out 2>/dev/null
  for K in 1 2; do timeout 300 python scripts/dsgd_emulate.py --parts $P --schedule ring --tokens $K --runs >> $out 2>/dev/null; done
done
timeout 300 python scripts/dsgd_emulate.py --parts 8 --runs --config yahoo >> $out 2>/dev/null
timeout 300 python scripts/dsgd_emulate.py --parts 8 --schedule ring --tokens 1 --runs --config yahoo >> $out 2>/dev/null
timeout 300 python scripts/dsgd_emulate.py --parts 1 --config yahoo >> $out 2>/dev/null
timeout 300 python scripts/dsgd_emulate.py --parts 1 >> $out 2>/dev/null
grep parts $out | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l)
    print(d['parts'], d['schedule'], d.get('tokens'), d.get('runs'), d['rank_nnz'], round(d['factor_ms'], 3), round(d['core_ms'], 3), round(d['epoch_ms'], 3), '%.3g' % d['implied_job_nnz_per_s'])"
