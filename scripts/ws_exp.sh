#!/bin/bash
# Timing experiments of the WS sweeps (FTKCU_WS_EXP bits; never production):
# 2 = no gathers, 16 = no factor write-back.
for e in ${EXPS:-0 2 16 18}; do FTKCU_WS_EXP=$e bash scripts/bench_brief.sh "$@" | sed "s/^/exp=$e /"; done
