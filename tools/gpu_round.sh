#!/bin/bash
# One gpurun session: smoke, tests, bench lines, ncu launch list of the default
# bench command, ncu --set full captures, FP64 census of the other configs.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --precision fp32 --no-cpu-baseline > gpurun_out/bench_cfg5_fp32.json 2> gpurun_out/bench_cfg5_fp32.err
for c in cfg1 cfg2 cfg3 cfg4; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
# launch list of the default bench command (serialised, cold-cache per launch)
CMD="python bench.py --steps 2 --warmup 3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg5.csv $CMD > gpurun_out/ncu_launch.log 2>&1
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,smsp__sass_thread_inst_executed_op_fp32_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
# full captures at 2^20 paths: without the draw store (the regime of 91% of
# cfg5's chunks on one GPU) and with it (cfg3 default)
PCMD="python tools/profile_case.py --config cfg3 --paths 1048576"
LTG_ZSTORE=0 $PCMD > gpurun_out/plain_profile_noz.log 2>&1 && \
  LTG_ZSTORE=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:heston_pass -c 2 \
    --metrics $M -o gpurun_out/prof_cfg3_noz -f $PCMD > gpurun_out/ncu_full_noz.log 2>&1
$PCMD > gpurun_out/plain_profile.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:heston_pass -c 2 \
    --metrics $M -o gpurun_out/prof_cfg3_full -f $PCMD > gpurun_out/ncu_full.log 2>&1
for spec in "cfg1 65536 fp64" "cfg2 262144 fp64" "cfg4 262144 fp64" "cfg3 262144 fp32"; do
  set -- $spec
  P2="python tools/profile_case.py --config $1 --paths $2 --precision $3"
  $P2 > gpurun_out/plain_$1_$3.log 2>&1 && \
    timeout 600 ncu --clock-control none -k regex:pass -c 2 --metrics $M --csv \
      --log-file gpurun_out/census_$1_$3.csv $P2 > gpurun_out/ncu_census_$1_$3.log 2>&1
done
ls gpurun_out
