#!/bin/bash
# ncu of the ring factor kernel (K = 1, cells in mode-3 runs) and of one
# strata cell sweep at P = 8 (Netflix shape, one GPU emulating rank 0).
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ws_factor -s 1 -c 1 -f \
  -o gpurun_out/ring_k1 python scripts/dsgd_emulate.py --parts 8 --schedule ring --tokens 1 --runs \
  --steps 1 --warmup 1 > gpurun_out/ring_k1.log 2>&1
echo "ring rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ws_factor -s 200 -c 1 -f \
  -o gpurun_out/strata_cell python scripts/dsgd_emulate.py --parts 8 --runs --steps 1 --warmup 1 \
  > gpurun_out/strata_cell.log 2>&1
echo "strata rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/strata_launches.csv python scripts/dsgd_emulate.py --parts 8 --runs \
  --steps 1 --warmup 1 > /dev/null 2>&1
echo "launches rc=$?"
