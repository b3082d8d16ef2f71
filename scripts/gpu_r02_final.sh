#!/bin/bash
# Round-2 evidence in one pass: GPU tests, smoke, default bench line (with
# CPU baseline, e2e, RMSE vs reference, fp32-equivalent), the reference arm,
# ncu launch list + full captures of the two headline sweeps at the Netflix
# and Yahoo shapes, the config sweep and the DSGD emulation.
tag=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
bash scripts/gpu_evidence.sh ${tag}_final > /dev/null 2>&1
rm -f gpurun_out/sweep_${tag}.jsonl; bash scripts/config_sweep.sh ${tag} > /dev/null 2>&1
bash scripts/dsgd_table.sh > /dev/null 2>&1; cp gpurun_out/dsgd_table.jsonl gpurun_out/${tag}_dsgd_emu.jsonl
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
