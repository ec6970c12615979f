"""Per-phase timeline of the fused decode kernel (dev tool, needs a GPU).

python tools/trace_decode.py [cfg4] [reps] [fused(1)|unfused(0)]
Prints, per stamp, the median / max over CTAs of (stamp - kernel start) in
microseconds (hata_debug_trace(), %globaltimer), stamps sorted by median.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402

NAMES = {31: "kernel_entry", 0: "start", 1: "hash_done", 2: "score_done", 3: "hist_x", 4: "D_staged", 5: "select_done",
         6: "attn_done", 7: "end(last)", 8: "qk_loaded", 9: "W_ready", 10: "stage0", 11: "thr",
         12: "quota", 13: "last_stage", 14: "unused14", 15: "published", 16: "kv_gathered",
         17: "groups_done", 19: "kv_issued", 20: "kv_gathered_1st", 21: "groups_done_1st",
         23: "kv_issued_1st", 20: "attn_entry", 24: "c_fenced", 25: "c_copy_issued", 26: "c_copied"}


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    fused = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
    sh = synth.CONFIGS[cfg]
    dev = torch.device("cuda", 0)
    sets = [bench.Step(sh, 2000 + i, dev) for i in range(8)]
    H = sets[0].H
    M = H.decode_ranks(sh.B, sh.Hq, sh.Hkv, sh.d, sh.rbits, sh.N, sh.k, sets[0].K.dtype)
    nct = M * sh.B * sh.Hkv
    buf = torch.zeros(nct * 32, dtype=torch.int64, device=dev)
    for s in sets:
        s.run()
    torch.cuda.synchronize()
    H._lib.check(H.lib().hata_debug_trace(buf.data_ptr()), "trace")
    print(f"{cfg}: M={M} ranks x {sh.B * sh.Hkv} units = {nct} CTAs  ({'fused' if fused else 'decode only'})")
    marks = torch.zeros(2, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    for rep in range(reps):
        s = sets[rep % len(sets)]
        buf.zero_()
        H.lib().hata_debug_timestamp(marks.data_ptr(), st)            # previous kernel done
        (s.run if fused else s.decode)()
        H.lib().hata_debug_timestamp(marks.data_ptr() + 8, st)        # decode kernel done
        torch.cuda.synchronize()
        t = buf.view(nct, 32).cpu().double()
        mk = marks.cpu().double()
        t0 = mk[0]
        print(f"rep{rep} marker_before=0  decode_done_marker={(mk[1] - t0).item() / 1e3:.2f} us")
        cols = []
        for i in range(32):
            c = t[:, i]
            c = c[c > 0]
            if len(c):
                c = (c - t0) / 1e3
                cols.append((c.median().item(), c.max().item(), NAMES.get(i, str(i))))
        cols.sort()
        print(f"rep{rep} " + " ".join(f"{nm}={md:.2f}/{mx:.2f}" for md, mx, nm in cols))
    H._lib.check(H.lib().hata_debug_trace(None), "trace off")


if __name__ == "__main__":
    main()
