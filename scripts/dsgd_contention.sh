#!/bin/bash
# DSGD per-rank cost breakdown (experiments build: FTKCU_WS_EXP=16 drops the
# factor write-back) and the RED rate on small tables (DSGD mode-3 blocks).
cd scripts/microtests && ./red_segments > ../../gpurun_out/red_segments_small.txt 2>&1; cd ../..
make -C paper_2404_10087_b200 clean >/dev/null; make -j8 -C paper_2404_10087_b200 EXPERIMENTS=1 >/dev/null 2>&1
for e in 0 16; do for sch in strata ring; do
  FTKCU_WS_EXP=$e timeout 300 python scripts/dsgd_emulate.py --parts 8 --schedule $sch 2>/dev/null | sed "s/^/exp=$e /"
done; done
make -C paper_2404_10087_b200 clean >/dev/null; make -j8 -C paper_2404_10087_b200 >/dev/null 2>&1
cat gpurun_out/red_segments_small.txt
