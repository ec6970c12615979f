#!/bin/bash
# Round-end evidence: GPU tests, bench line, ncu launch list + full captures
# (decode and prefill hash), smoke, phase trace.  usage: tools/final_check.sh TAG
TAG=${1:-final}
NCU=1 bash tools/gpu_check.sh $TAG
timeout 400 ncu --set full --clock-control none --import-source on -k regex:hash_keys_mma -c 1 -o gpurun_out/prof_hash_$TAG python bench.py --steps 10 --warmup 3 --no-cpu --no-secondary > gpurun_out/ncu_hash_$TAG.log 2>&1
tail -1 gpurun_out/ncu_hash_$TAG.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
timeout 120 python tools/trace_decode.py cfg4 3 1 > gpurun_out/trace_$TAG.txt 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; cat gpurun_out/bench_ref_$TAG.json
