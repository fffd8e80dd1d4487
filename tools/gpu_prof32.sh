#!/bin/bash
# ncu full capture of both Heston passes on cfg3 in fp32 mode (argument: tag, paths)
TAG=${1:-f32}; P=${2:-262144}
PCMD="python tools/profile_case.py --config cfg3 --paths $P --precision fp32"
$PCMD > gpurun_out/plain_profile32.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:heston_pass -c 2 \
    -o gpurun_out/prof_$TAG -f $PCMD > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
