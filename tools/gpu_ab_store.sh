#!/bin/bash
# A/B timing with the draw store on (cfg3 / cfg2 defaults: every chunk's draws
# stored) of the main build and the named variants. usage: tools/gpu_ab_store.sh name...
for v in main "$@" main "$@"; do
  lib=""; [ "$v" != main ] && lib=paper_1901_04200_b200/_lib/variants/$v.so
  env ${lib:+LTG_LIB=$lib} timeout 200 python tools/quick_time.py ${QT_CFGS:-cfg3 cfg3:fp32 cfg2} 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try:
        d = json.loads(l); print('$v', d['cfg'], 'p1 %.3f p2 %.3f tot %.3f' % (d['pass1_ms'], d['pass2_ms'], d['total_ms']))
    except Exception: print('$v', l.strip()[:200])"
done
