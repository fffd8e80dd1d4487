#!/bin/bash
# One gpurun session: smoke, tests, bench lines, ncu launch list + full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
for c in cfg1 cfg2 cfg3; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
# ncu: launch list of a short cfg3 bench, then the full capture of both passes at 2^18 paths
CMD="python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_cfg3.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv $CMD > gpurun_out/ncu_launch.log 2>&1
PCMD="python tools/profile_case.py --config cfg3 --paths 262144"
$PCMD > gpurun_out/plain_profile.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:heston_pass -c 2 \
    --metrics smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum \
    -o gpurun_out/prof_cfg3 -f $PCMD > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
