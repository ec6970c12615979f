for r in 1 2 3; do
 for cfg in "libhata_prev.so 1" "libhata.so 1" "libhata.so 0"; do set -- $cfg
  HATA_LIB=$1 HATA_BENCH_COOP=$2 timeout 200 python bench.py --no-cpu --no-secondary --steps 1600 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 coop=$2', 'us', round(d['us_per_step'],3), 'e2e', round(d['e2e']['us_per_step'],2))"
 done
done
HATA_LIB=libhata.so timeout 300 python -m pytest tests/test_gpu_paths.py -q -x -k "bench_launch or ragged" 2>&1 | tail -1
HATA_BENCH_COOP=0 HATA_LIB=libhata_trace_hot.so timeout 120 python tools/trace_decode.py chain cfg4 > gpurun_out/trace_s4_nc.txt 2>&1; tail -3 gpurun_out/trace_s4_nc.txt | cut -c1-1400
