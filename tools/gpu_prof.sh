#!/bin/bash
# ncu full capture of both Heston passes on cfg3 (argument: tag, paths)
TAG=${1:-cur}; P=${2:-262144}
PCMD="python tools/profile_case.py --config cfg3 --paths $P"
M=smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum
$PCMD > gpurun_out/plain_profile.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:heston_pass -c 2 \
    --metrics $M -o gpurun_out/prof_$TAG -f $PCMD > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
