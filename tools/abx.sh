#!/bin/bash
# A/B of decode builds on one box.  usage: tools/abx.sh TAG LIB[:TRACELIB] ...
# LIB is a file name under paper_2506_02572_b200/ (libhata.so = product).
# Per build: a parity subset (CFG-4-shaped tests), the bench decode line 3x
# alternating with the other builds, and one phase trace if TRACELIB is given.
TAG=$1; shift
mkdir -p gpurun_out
for VS in "$@"; do
  L=${VS%%:*}
  echo "== parity $L"
  HATA_LIB=$L timeout 400 python -m pytest tests/test_gpu_paths.py tests/test_gpu_parity.py -q -x \
     -k "bench_launch or ragged or kv_pair and cfg4 or full_size and cfg4 or hinted and cfg2 or stale" 2>&1 | tail -2
done
for round in 1 2 3; do
  for VS in "$@"; do
    L=${VS%%:*}
    HATA_LIB=$L timeout 200 python bench.py --no-cpu --no-secondary --steps 1600 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', 'us', round(d['us_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['us_per_step'],2), d.get('hint', ''))"
  done
done
for VS in "$@"; do
  case $VS in *:*) T=${VS#*:}; HATA_LIB=$T timeout 120 python tools/trace_decode.py cfg4 3 1 > gpurun_out/trace_${TAG}_${T%.so}.txt 2>&1; HATA_LIB=$T timeout 120 python tools/trace_decode.py chain cfg4 >> gpurun_out/trace_${TAG}_${T%.so}.txt 2>&1
     echo "== trace $T"; grep 'rep2 \|launch' gpurun_out/trace_${TAG}_${T%.so}.txt | tail -6 | cut -c1-1500;;
  esac
done
