#!/bin/bash
# One GPU round: parity tests, bench, ncu launch list + full capture of the decode kernel.
# usage: tools/gpu_check.sh TAG [pytest-k-expr]
TAG=${1:-x}
KEXPR=${2:-"not full_size_batched"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x -k "$KEXPR" > gpurun_out/pytest_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_$TAG.log
tail -15 gpurun_out/pytest_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
if [ -n "$NCU" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hata -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-secondary > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:hata_decode -s 40 -c 1 -o gpurun_out/prof_decode_$TAG python bench.py --steps 10 --warmup 3 --no-cpu --no-secondary > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
fi
