#!/bin/bash
# A/B timing of the main build and the variants named on the command line
# (paper_1901_04200_b200/_lib/variants/<name>.so): cfg3 fp64 / fp32 passes
# without the draw store, then the cfg5 bench line of each precision.
# usage: tools/gpu_ab.sh [--cfg5] name...
CFG5=0; [ "$1" = "--cfg5" ] && { CFG5=1; shift; }
for v in main "$@"; do
  lib=""; [ "$v" != main ] && lib=paper_1901_04200_b200/_lib/variants/$v.so
  for rep in 1 2; do
    env LTG_ZSTORE=0 ${lib:+LTG_LIB=$lib} timeout 200 python tools/quick_time.py ${QT_CFGS:-cfg3 cfg3:fp32 cfg4 cfg2} 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try:
        d = json.loads(l); print('$v', d['cfg'], 'p1 %.3f p2 %.3f tot %.3f' % (d['pass1_ms'], d['pass2_ms'], d['total_ms']))
    except Exception: print('$v', l.strip()[:200])"
  done
  if [ $CFG5 = 1 ]; then
    for prec in fp64 fp32; do
      env ${lib:+LTG_LIB=$lib} timeout 300 python bench.py --no-cpu-baseline --precision $prec --steps 3 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v cfg5 $prec %.4g paths/s' % d['value'], d['pass_ms'], 'frac', round(d['roofline']['frac'], 3))"
    done
  fi
done
