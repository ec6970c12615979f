for d in 0 2 16 18; do
HATA_DEBUG=$d HATA_LIB=libhata_trace.so timeout 120 python tools/trace_decode.py cfg4 3 1 > gpurun_out/trace_dbg$d.txt 2>&1
echo "dbg=$d"; grep 'rep2 kernel_entry' gpurun_out/trace_dbg$d.txt | tr ' ' '\n' | grep -E 'stage0|last_stage|score_done|hash_done'  | tr '\n' ' '; echo
done
