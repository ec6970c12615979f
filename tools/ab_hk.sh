#!/bin/bash
# Same-box A/B of the prefill hash (hash_keys) and decode timings per library.
for round in 1 2; do
  for lib in "$@"; do
    HATA_LIB=$lib timeout 120 python bench.py --no-cpu --no-secondary --steps 200 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('round $round $lib decode', round(d['us_per_step'],2), 'hash_keys', round(d['hash_keys']['us'],1), 'us', round(d['hash_keys']['TFLOPs'],1), 'TFLOP/s')"
  done
done
