#!/bin/bash
# quick GPU check: parity subset + trace + bench (+ optional HATA_DEBUG variants in $DBGS)
timeout 900 python -m pytest tests/ -q -m gpu -x -k "not full_size_batched and not shard" 2>&1 | grep -E "passed|failed|error" | sed "s/^/pytest: /"
python tools/trace_decode.py cfg4 3 1 2>&1 | tail -2
for d in 0 $DBGS; do
  echo -n "dbg=$d bench: "
  HATA_DEBUG=$d timeout 600 python bench.py --no-cpu --no-secondary --steps 400 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['us_per_step'],2), round(d['roofline']['frac'],4), round(d['e2e']['us_per_step'],2))"
done
