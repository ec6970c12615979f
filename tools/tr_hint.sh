for h in 1 0; do
HATA_HINT=$h HATA_LIB=libhata_trace.so timeout 120 python tools/trace_decode.py cfg4 3 1 > gpurun_out/trace_s2m_h$h.txt 2>&1
echo "hint=$h"; grep 'rep2 kernel_entry' gpurun_out/trace_s2m_h$h.txt
done
