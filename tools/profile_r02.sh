#!/bin/bash
# Round-2 evidence: ncu launch list of the bench's decode launches, one
# --set full capture each of the decode kernel, the tcgen05 hash kernel and
# the fused prefill write, and the chained phase trace.  1 GPU.
mkdir -p gpurun_out
T=${1:-r02}
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hata_decode -s 64 -c 64 --csv \
  --log-file gpurun_out/launches_$T.csv python bench.py --steps 64 --warmup 16 --no-cpu --no-secondary > /dev/null 2>&1
echo launches $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hata_decode -s 80 -c 1 \
  -o gpurun_out/prof_decode_$T python bench.py --steps 64 --warmup 16 --no-cpu --no-secondary > gpurun_out/ncu_dec_$T.log 2>&1
echo decode $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hash_keys_umma -c 2 \
  -o gpurun_out/prof_hash_$T python bench.py --steps 16 --warmup 3 --no-cpu --no-secondary > gpurun_out/ncu_hash_$T.log 2>&1
echo hash $?
HATA_TRACE_BUILD=1 python -m paper_2506_02572_b200.build > /dev/null 2>&1
HATA_LIB=libhata_trace.so timeout 300 python tools/trace_decode.py chain cfg4 > gpurun_out/trace_chain_$T.txt 2>&1
echo trace $?
