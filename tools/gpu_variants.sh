#!/bin/bash
mkdir -p gpurun_out
for v in paper_1901_04200_b200/_lib/variants/*.so; do
  echo "== $v"; LTG_LIB=$v timeout 120 python tools/quick_time.py cfg3 cfg2 2>&1 | tail -2 | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['cfg'], 'p1 %.2f p2 %.2f tot %.2f' % (d['pass1_ms'], d['pass2_ms'], d['total_ms']))"
done
PCMD="python tools/profile_case.py --config cfg3 --paths 262144"
$PCMD > gpurun_out/plain_profile.log 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:heston_pass -c 2 \
    --metrics smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_fp64_pred_on.sum \
    -o gpurun_out/prof_cfg3_v2 -f $PCMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
