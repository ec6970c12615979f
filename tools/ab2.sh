#!/bin/bash
# Same-box A/B of bench timings: each arg is LIB[:ENV=VAL,...]; 3 alternating rounds.
for round in 1 2 3; do
  for spec in "$@"; do
    lib=${spec%%:*}; envs=""; [ "$spec" != "$lib" ] && envs=${spec#*:}
    r=$(env ${envs//,/ } HATA_LIB=$lib timeout 120 python bench.py --no-cpu --no-secondary --steps 400 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],2))" 2>/dev/null)
    echo "round $round $spec: $r"
  done
done
