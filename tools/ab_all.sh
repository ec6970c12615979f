#!/bin/bash
# Same-box A/B of whole bench lines (cfg4 + secondary) for several libraries
for round in 1 2; do
  for lib in "$@"; do
    HATA_LIB=$lib timeout 600 python bench.py --no-cpu --steps 200 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('round $round $lib cfg4', round(d['us_per_step'],2), round(d['roofline']['frac'],4), *[(k, round(v['us_per_step'],2), round(v['frac'],4)) for k,v in d['secondary'].items()])"
  done
done
