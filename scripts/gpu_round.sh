#!/bin/bash
# Round evidence in one GPU-box pass: GPU tests, smoke, default bench line,
# ncu launch list of the bench command, full ncu captures of the two headline
# sweeps, and a bench line per BASELINE config.
tag=${1:-r01}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/b_ncu.log 2>&1
for k in ws_factor ws_core16; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -f -o gpurun_out/${tag}_$k python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${tag}_$k.log 2>&1
done
rm -f gpurun_out/sweep_${tag}.jsonl
bash scripts/config_sweep.sh ${tag}
timeout 600 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 --store-c 1 2>/dev/null | tail -1 >> gpurun_out/sweep_${tag}.jsonl
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/bench.json gpurun_out/bench_ref.json
