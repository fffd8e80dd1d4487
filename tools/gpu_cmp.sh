#!/bin/bash
# GPU tests, then cfg3 (draw store on/off) and cfg5 bench for the main build and every variant
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in "" paper_1901_04200_b200/_lib/variants/*.so; do
  [ -n "$v" ] && [ ! -f "$v" ] && continue
  for env in "LTG_ZSTORE=1" "LTG_ZSTORE=0"; do
    echo "== ${v:-main} $env"; env $env ${v:+LTG_LIB=$v} timeout 120 python tools/quick_time.py cfg3 2>&1 | tail -1 | python -c "
import sys, json
for l in sys.stdin:
    try:
        d = json.loads(l); print(d['cfg'], 'p1 %.2f p2 %.2f tot %.2f' % (d['pass1_ms'], d['pass2_ms'], d['total_ms']))
    except Exception: print(l.strip()[:200])"
  done
  echo "== ${v:-main} cfg5"; env ${v:+LTG_LIB=$v} timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5 %.4g paths/s' % d['value'], d['pass_ms'], 'frac', round(d['roofline']['frac'], 3))"
done
