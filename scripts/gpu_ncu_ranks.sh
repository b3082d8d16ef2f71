#!/bin/bash
# ncu --set full of the dominant sweeps at J = R = 64 and 128 (Netflix shape)
# and at J = R = 8 / 16 (WSG), summaries into gpurun_out/.
mkdir -p gpurun_out
for r in 64 128; do
  for k in big_factor big_core big128_factor big16p_core big16_core; do :; done
done
run() {  # rank, kernel regex, tag
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 \
    -f -o gpurun_out/r02_j$1_$3 python bench.py --rank $1 --steps 1 --warmup 1 \
    --no-cpu --no-e2e --no-rmse-check --no-fp32-equiv > gpurun_out/r02_j$1_$3.log 2>&1
  echo "J=$1 $3 rc=$?"
  python scripts/ncu_summary.py gpurun_out/r02_j$1_$3.ncu-rep 20 > gpurun_out/r02_j$1_$3_summary.txt 2>&1
}
run 64 "big.*factor" factor
run 64 "big.*core" core
run 128 "big.*factor" factor
run 128 "big.*core" core
run 8 "wsg_factor" factor
run 16 "wsg_factor" factor
