#!/bin/bash
# A/B of decode builds on one box.  usage: tools/abx.sh TAG LIB[:TRACELIB] ...
# LIB is a file name under paper_2506_02572_b200/ (libhata.so = product).
# Per build: a CFG-4 parity subset, the bench decode line 3x alternating with
# the other builds (q varying per replay), and one chained phase trace if
# TRACELIB is given.
TAG=$1; shift
mkdir -p gpurun_out
for VS in "$@"; do
  L=${VS%%:*}
  echo "== parity $L"
  HATA_LIB=$L timeout 400 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x \
     -k "bench_launch or ragged or kv_pair and cfg4 or full_size and cfg4 or hinted and cfg2 or stale" 2>&1 | tail -1
done
for round in 1 2 3; do
  for VS in "$@"; do
    L=${VS%%:*}
    HATA_LIB=$L timeout 200 python bench.py --no-cpu --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', 'us', round(d['us_per_step'],3), 'p5/p95', round(d['latency_us']['p5'],2), round(d['latency_us']['p95'],2), 'nohint', round(d['no_hint_us_per_step'],2), 'hint', round(d['selection_hint']['hinted_selection_rate'],2))"
  done
done
for VS in "$@"; do
  case $VS in *:*) T=${VS#*:}; HATA_LIB=$T timeout 120 python tools/trace_decode.py chain cfg4 > gpurun_out/trace_${TAG}_${T%.so}.txt 2>&1
     echo "== trace $T"; grep 'launch' gpurun_out/trace_${TAG}_${T%.so}.txt | tail -2 | cut -c1-1500;;
  esac
done
