#!/bin/bash
# One ncu --set full capture of the decode kernel in the bench configuration
# (1 GPU; never under a multi-rank command).  usage: tools/ncu_decode.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hata_decode -s 40 -c 1 \
  -o gpurun_out/prof_decode_$TAG python bench.py --steps 48 --warmup 3 --no-cpu --no-secondary > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
