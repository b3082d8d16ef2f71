#!/bin/bash
# DSGD ring: GPU tests (virtual ranks), per-rank emulation of both schedules
# at P = 2, 4, 8, and one ncu capture of the ring factor kernel (P = 8).
timeout 900 python -m pytest tests/test_dsgd_gpu.py -q -x -k "ring" > gpurun_out/ring_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ring_tests.log; tail -4 gpurun_out/ring_tests.log
rm -f gpurun_out/ring_emu.jsonl
for P in 2 4 8; do
  timeout 300 python scripts/dsgd_emulate.py --parts $P --schedule strata >> gpurun_out/ring_emu.jsonl 2>>gpurun_out/ring_emu.err
  for K in 1 2; do timeout 300 python scripts/dsgd_emulate.py --parts $P --schedule ring --tokens $K >> gpurun_out/ring_emu.jsonl 2>>gpurun_out/ring_emu.err; done
done
grep parts gpurun_out/ring_emu.jsonl | python -c "
import json
import sys
for l in sys.stdin:
    d=json.loads(l); print(d['parts'], d['schedule'], d.get('tokens'), round(d['factor_ms'],3), round(d['core_ms'],3), round(d['epoch_ms'],3), '%.3g'%d['implied_job_nnz_per_s'])"
if [ "${NCU:-1}" = 1 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ws_factor -s 1 -c 1 -f -o gpurun_out/ring_p8 python scripts/dsgd_emulate.py --parts 8 --schedule ring --steps 1 --warmup 1 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/ring_p8.ncu-rep 20 > gpurun_out/ring_p8_summary.txt 2>&1; head -14 gpurun_out/ring_p8_summary.txt
fi
