#!/bin/bash
# ncu full capture of the two passes of any config (arguments: tag config paths [precision])
TAG=$1; CFG=$2; P=$3; PREC=${4:-fp64}
PCMD="python tools/profile_case.py --config $CFG --paths $P --precision $PREC"
$PCMD > gpurun_out/plain_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:pass -c 2 \
    -o gpurun_out/prof_$TAG -f $PCMD > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
