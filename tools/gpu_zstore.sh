#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for env in "" "LTG_ZSTORE=0" "LTG_CKPT_STEPS=16" "LTG_CKPT_STEPS=16 LTG_ZSTORE=0"; do
  echo "== $env"; env $env timeout 300 python tools/quick_time.py cfg3 2>&1 | tail -1 | cut -c1-330
done
for env in "" "LTG_CKPT_STEPS=16"; do
  echo "== cfg5 $env"; env $env timeout 300 python bench.py --no-cpu-baseline --steps 3 2>&1 | tail -1 | python -c "
import sys, json; d = json.loads(sys.stdin.read()); print('%.4g' % d['value'], d['pass_ms'], d['config'].get('checkpoint_interval_steps'), d['roofline']['frac'])"
done
