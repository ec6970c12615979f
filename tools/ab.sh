#!/bin/bash
# A/B of experimental builds: for each variant V (libhata_V.so; "base" = libhata.so)
# run a parity subset, the bench (decode only) and, if libhata_trace_V.so exists, the phase trace.
# usage: tools/ab.sh TAG V1 V2 ...
TAG=$1; shift
mkdir -p gpurun_out
for VS in "$@"; do
  V=${VS%@*}; PDL=1; [ "$VS" != "$V" ] && PDL=${VS#*@}
  export HATA_PDL=$PDL
  if [ "$V" = base ]; then L=libhata.so; LT=libhata_trace.so; else L=libhata_$V.so; LT=libhata_trace_$V.so; fi
  echo "== $V pdl=$PDL"
  HATA_LIB=$L timeout 300 python -m pytest tests/ -q -m gpu -x -k "not full_size_batched and not shard" 2>&1 | grep -E "passed|failed|error|Error" | head -5 | sed "s/^/pytest: /"
  for i in 1 2; do
    HATA_LIB=$L timeout 120 python bench.py --no-cpu --no-secondary --steps 400 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['us_per_step'],2), round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['us_per_step'],2))"
  done
  if [ -f paper_2506_02572_b200/$LT ]; then
    HATA_LIB=$LT timeout 120 python tools/trace_decode.py cfg4 3 1 > gpurun_out/trace_${TAG}_${V}_$PDL.txt 2>&1
    grep 'rep2 kernel_entry' gpurun_out/trace_${TAG}_${V}_$PDL.txt | tr ' ' '\n' | head -40 | tr '\n' ' '; echo
    grep 'rep2 select cycles\|rep2 combine' gpurun_out/trace_${TAG}_${V}_$PDL.txt
  fi
done
