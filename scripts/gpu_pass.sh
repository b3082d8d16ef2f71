#!/bin/bash
# One GPU-box pass of selected steps (each bounded by its own timeout):
#   bash scripts/gpu_pass.sh "acc traj bench ref" [pytest-args]
steps=${1:-"acc bench"}
mkdir -p gpurun_out
for st in $steps; do
  case $st in
    acc)   timeout 1500 python -m pytest tests/test_accuracy_gpu.py -q -x > gpurun_out/acc.log 2>&1; echo "rc=$?" >> gpurun_out/acc.log; tail -3 gpurun_out/acc.log ;;
    gpu)   timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log ;;
    traj)  timeout 1800 python oracle/gen_c2_trajectory.py 3 > gpurun_out/traj.log 2>&1; echo "rc=$?" >> gpurun_out/traj.log; cp tests/golden/c2_trajectory.json gpurun_out/ 2>/dev/null; tail -3 gpurun_out/traj.log ;;
    bench) timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err ;;
    probe) timeout 1500 python scripts/c2_rmse_probe.py uniform "precision=1" "precision=1,max_ctas=37" "precision=1,max_ctas=4" "precision=1,hog_update=0" "precision=2" "precision=0" "precision=1,core16=0" "precision=1,core16=2" > gpurun_out/probe.jsonl 2> gpurun_out/probe.err; cat gpurun_out/probe.jsonl; tail -3 gpurun_out/probe.err ;;
    b3)    timeout 900 python bench.py --precision 3xtf32 --no-cpu --no-e2e --no-rmse-check > gpurun_out/bench3.json 2> gpurun_out/bench3.err; cat gpurun_out/bench3.json; tail -3 gpurun_out/bench3.err ;;
    bq)    timeout 900 python bench.py --no-cpu --no-e2e --no-rmse-check > gpurun_out/benchq.json 2> gpurun_out/benchq.err; cat gpurun_out/benchq.json; tail -3 gpurun_out/benchq.err ;;
    ref)   timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err ;;
  esac
done
