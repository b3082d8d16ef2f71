#!/bin/bash
# usage: scripts/bench_brief.sh [bench.py args...]  -> one-line summary
timeout 300 python bench.py --no-cpu --no-e2e "$@" 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('%s value=%.4g ms=%.2f phases=%s frac=%.3f loss=%s clocks=%s' % (' '.join(sys.argv[1:]), d['value'], d['ms_per_step'], {k: round(v,2) for k,v in d['phases_ms'].items()}, d['roofline']['frac'], [('%.4g' % x) for x in d['train_loss_before_after']], d['clocks']['sm_mhz']))
" "$@"
