#!/bin/bash
# Build the product library and the diagnostics build in parallel; fail loudly.
cd "$(dirname "$0")/.."
python -m paper_2506_02572_b200.build --force > /tmp/build_prod.log 2>&1 & P1=$!
HATA_TRACE_BUILD=1 python -m paper_2506_02572_b200.build --force > /tmp/build_trace.log 2>&1 & P2=$!
wait $P1; R1=$?; wait $P2; R2=$?
if [ $R1 -ne 0 ] || [ $R2 -ne 0 ]; then tail -n 20 /tmp/build_prod.log /tmp/build_trace.log; echo BUILD FAILED; exit 1; fi
echo BUILD OK
