#!/bin/bash
# Same-box A/B of the K/V cache layout (pair vs split), decode + secondary configs
for round in 1 2; do
  for lay in split pair; do
    HATA_KV_LAYOUT=$lay timeout 600 python bench.py --no-cpu --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('round $round $lay cfg4', round(d['us_per_step'],2), round(d['roofline']['frac'],4), *[(k, round(v['us_per_step'],2), round(v['frac'],4)) for k,v in d['secondary'].items()], 'dense', round(d['dense_baseline']['us_per_step'],1))"
  done
done
