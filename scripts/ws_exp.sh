#!/bin/bash
# Timing experiments of the WS sweeps (FTKCU_WS_EXP bits; never production).
for e in 0 1 2 4 8 12 14; do FTKCU_WS_EXP=$e bash scripts/bench_brief.sh "$@" | sed "s/^/exp=$e /"; done
