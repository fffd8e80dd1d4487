#!/bin/bash
for v in "" paper_1901_04200_b200/_lib/variants/*.so; do
  for env in "LTG_ZSTORE=1" "LTG_ZSTORE=0"; do
  echo "== $v $env"; env $env ${v:+LTG_LIB=$v} timeout 120 python tools/quick_time.py cfg3 2>&1 | tail -1 | python -c "
import sys, json
for l in sys.stdin:
    try:
        d = json.loads(l); print(d['cfg'], 'p1 %.2f p2 %.2f tot %.2f' % (d['pass1_ms'], d['pass2_ms'], d['total_ms']))
    except Exception: print(l.strip()[:200])"
  done
done
