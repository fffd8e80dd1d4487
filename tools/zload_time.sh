#!/bin/bash
# pass-2 time with the draw store (cfg3 2^20; config 5's per-GPU share at 8 GPUs) for every build
for v in "" paper_1901_04200_b200/_lib/variants/*.so; do
  [ -n "$v" ] && [ ! -f "$v" ] && continue
  echo "== ${v:-main}"; env ${v:+LTG_LIB=$v} timeout 120 python tools/quick_time.py cfg3 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print('cfg3 p1 %.2f p2 %.2f' % (d['pass1_ms'], d['pass2_ms']))"
  env ${v:+LTG_LIB=$v} timeout 300 python bench.py --paths 8388608 --no-cpu-baseline --no-alt-method 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('2^23', d['pass_ms'])"
done
