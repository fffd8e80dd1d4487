#!/bin/bash
# cfg5 tangent-mode time for the main build and every variant
for v in "" paper_1901_04200_b200/_lib/variants/*.so; do
  [ -n "$v" ] && [ ! -f "$v" ] && continue
  echo "== ${v:-main}"; env ${v:+LTG_LIB=$v} timeout 300 python bench.py --method tangent --no-cpu-baseline --no-alt-method 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('tangent %.4g paths/s' % d['value'], d['pass_ms'])"
done
