#!/bin/bash
# Round evidence on one B200: bench line, launch list, full ncu captures of the
# two hot sweeps at the Netflix and Yahoo shapes, summaries.
#   bash scripts/gpu_evidence.sh TAG
tag=${1:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -1 gpurun_out/${tag}_bench.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e \
  --no-rmse-check --no-fp32-equiv > /dev/null 2>&1
echo "launches rc=$?"
for cfg in netflix yahoo; do
  for k in ws_factor ws_core16; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -f -o gpurun_out/${tag}_${cfg}_$k python bench.py --config $cfg --steps 1 --warmup 1 \
      --no-cpu --no-e2e --no-rmse-check --no-fp32-equiv > gpurun_out/${tag}_${cfg}_$k.log 2>&1
    echo "$cfg $k rc=$?"
    python scripts/ncu_summary.py gpurun_out/${tag}_${cfg}_$k.ncu-rep 20 > gpurun_out/${tag}_${cfg}_${k}_summary.txt 2>&1
    python scripts/ncu_top.py gpurun_out/${tag}_${cfg}_$k.ncu-rep 25 > gpurun_out/${tag}_${cfg}_${k}_top.txt 2>&1
  done
done
