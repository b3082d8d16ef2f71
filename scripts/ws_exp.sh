#!/bin/bash
# Timing experiments of the WS sweeps (FTKCU_WS_EXP bits; never production):
# 2 = no gathers, 16 = no factor write-back.  Needs an experiments build:
#   make -C paper_2404_10087_b200 clean all EXPERIMENTS=1   (rebuild without it after)
for e in ${EXPS:-0 2 16 18}; do FTKCU_WS_EXP=$e bash scripts/bench_brief.sh "$@" | sed "s/^/exp=$e /"; done
