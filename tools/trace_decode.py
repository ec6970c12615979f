"""Per-phase timeline of the fused decode kernel (dev tool, needs a GPU).

python tools/trace_decode.py [cfg4] [reps] [fused(1)|unfused(0)]
Prints, per stamp, the median / max over CTAs of (stamp - kernel start) in
microseconds (hata_debug_trace(), %globaltimer), stamps sorted by median.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

os.environ.setdefault("HATA_LIB", "libhata_trace.so")   # the build with the phase stamps compiled in

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402

NAMES = {31: "kernel_entry", 0: "start", 1: "hash_done", 2: "score_done", 3: "hist_x", 4: "merge_ml_polled", 5: "select_done",
         6: "attn_done", 7: "end(last)", 8: "qk_loaded", 9: "W_ready", 10: "stage0", 11: "thr",
         12: "merge_out_polled", 13: "last_stage", 14: "merge_polled", 15: "published", 16: "kv_gathered",
         17: "groups_done", 19: "kv_issued", 20: "kv_gathered_1st", 21: "groups_done_1st",
         23: "kv_issued_1st", 20: "attn_entry", 27: "arrived", 28: "wait_done", 18: "sel_counted", 21: "sel_scanned", 22: "sel_emitted", 29: "attn_wmerge1", 30: "attn_wmerge2", 24: "hash_mma_done(t0)", 25: "hash_synced", 26: "planes_done(t0)"}


def chain(cfg, S=8):
    """S fused steps over S cache sets captured in ONE CUDA graph (the bench's
    launch configuration, PDL between steps), each launch with its own trace
    buffer: stamps of launch i are reported relative to the end of launch
    i-1 (the max 'end(last)' stamp of its merging CTAs)."""
    sh = synth.CONFIGS[cfg]
    dev = torch.device("cuda", 0)
    bench.apply_options()
    sets = [bench.Step(sh, 2000 + i, dev) for i in range(S)]
    H = sets[0].H
    M = H.decode_ranks(sh.B, sh.Hq, sh.Hkv, sh.d, sh.rbits, sh.N, sh.k, sets[0].K.dtype)
    nct = M * sh.B * sh.Hkv
    bufs = [torch.zeros(nct * 96, dtype=torch.int64, device=dev) for _ in range(S)]

    def run_all():
        for s, b in zip(sets, bufs):
            H._lib.check(H.lib().hata_debug_trace(b.data_ptr()), "trace")
            s.run()
        H._lib.check(H.lib().hata_debug_trace(None), "trace off")
    g = bench._graph(run_all)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for b in bufs:
        b.zero_()
    g.replay()
    torch.cuda.synchronize()
    ts = [b.view(nct, 96).cpu().double() for b in bufs]
    print(f"{cfg} chained x{S}: M={M} ranks x {sh.B * sh.Hkv} units = {nct} CTAs")
    for i in range(1, S):
        prev_end = ts[i - 1][:, 7].max()
        t = ts[i]
        cols = []
        for j in range(32):
            c = t[:, j]
            c = c[c > 0]
            if len(c):
                c = (c - prev_end) / 1e3
                cols.append((c.median().item(), c.max().item(), NAMES.get(j, str(j))))
        cols.sort()
        step = (t[:, 7].max() - prev_end) / 1e3
        print(f"launch{i} step={step.item():.2f}us " + " ".join(f"{nm}={md:.2f}/{mx:.2f}" for md, mx, nm in cols))
        if i == S - 1:
            # clock-refined timeline: each stamp = the CTA's wait_done (globaltimer,
            # 256 ns ticks) + (clock64 delta) / (its own clock rate over the launch)
            ck = t[:, 64:96]
            ok = (t[:, 28] > 0) & (t[:, 31] > 0)
            span_gt = t[:, 15].where(t[:, 15] > 0, t[:, 7]) - t[:, 31]
            span_ck = ck[:, 15].where(t[:, 15] > 0, ck[:, 7]) - ck[:, 31]
            f = (span_ck / span_gt.clamp(min=1)).median().item()       # cycles per ns
            fine = []
            for j in range(32):
                sel = ok & (t[:, j] > 0)
                if sel.any():
                    v = ((t[sel, 28] - prev_end) + (ck[sel, j] - ck[sel, 28]) / f) / 1e3
                    fine.append((v.median().item(), v.max().item(), NAMES.get(j, str(j))))
            CLKN = {17: "q_rows_loaded(t0)", 18: "sync_words_loaded", 19: "hash_qa_loaded", 20: "hash_mma_chain_done",
                    21: "hash_planes_w0", 22: "prefix_scanned", 24: "counts_published", 25: "fsel_words_done",
                    26: "fsel_scanned", 27: "fsel_quota", 29: "merge_weights(t0)", 30: "merge_outputs_done",
                    11: "stage0_landed", 12: "stage1_landed", 13: "stage2_landed"}
            for j, nm in CLKN.items():
                sel = ok & (t[:, 32 + j] > 0)
                if sel.any():
                    v = ((t[sel, 28] - prev_end) + (t[sel, 32 + j] - ck[sel, 28]) / f) / 1e3
                    fine.append((v.median().item(), v.max().item(), "c:" + nm))
            fine.sort()
            print(f"  clock-refined ({f:.3f} GHz):")
            for md, mx, nm in fine:
                print(f"    {md:7.2f} {mx:7.2f}  {nm}")
            # per rank (median over the units): when it reached each phase, and its selected rows
            rk = torch.arange(nct) % M
            for rr in range(M):
                sel = rk == rr
                row = []
                for j in (27, 3, 11, 22, 19, 16, 17, 6, 15, 4, 12, 14, 7):
                    c = t[sel, j]
                    c = c[c > 0]
                    if len(c):
                        row.append(f"{NAMES.get(j, j)}={((c - prev_end) / 1e3).median().item():.2f}")
                rows_sel = t[sel, 32 + 15]
                sp = t[sel, 32 + 16]
                used = (sp >= 100000).double().mean().item()
                cands = sp % 100000
                print(f"  rank{rr:2d} rows={rows_sel.median().item():.0f}/{rows_sel.max().item():.0f} "
                      f"spec={cands.median().item():.0f}/{cands.max().item():.0f} used={used:.2f} " + " ".join(row))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "chain":
        chain(sys.argv[2] if len(sys.argv) > 2 else "cfg4")
        return
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    fused = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
    sh = synth.CONFIGS[cfg]
    dev = torch.device("cuda", 0)
    sets = [bench.Step(sh, 2000 + i, dev) for i in range(int(os.environ.get('TRACE_SETS', '8')))]
    H = sets[0].H
    M = H.decode_ranks(sh.B, sh.Hq, sh.Hkv, sh.d, sh.rbits, sh.N, sh.k, sets[0].K.dtype)
    nct = M * sh.B * sh.Hkv
    buf = torch.zeros(nct * 96, dtype=torch.int64, device=dev)
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
        t = buf.view(nct, 96).cpu().double()
        mk = marks.cpu().double()
        t0 = mk[0]
        print(f"rep{rep} marker_before=0  decode_done_marker={(mk[1] - t0).item() / 1e3:.2f} us")
        cols = []
        last = (t[:, 7] > 0)
        if last.any():
            cyc = (t[last, 32 + 14] - t[last, 32 + 23]).median().item()
            ns = (t[last, 7] - t[last, 31]).median().item()
            print(f"rep{rep} clock: {cyc:.0f} cycles over {ns:.0f} ns -> {cyc / max(ns, 1):.3f} GHz (last ranks)")
        for i in range(32):
            pass
            c = t[:, i]
            c = c[c > 0]
            if len(c):
                c = (c - t0) / 1e3
                cols.append((c.median().item(), c.max().item(), NAMES.get(i, str(i))))
        cols.sort()
        ck = t[:, 32:]
        names = ["count_start", "count_loop", "warp_sums", "quota(bl/ti)", "sync", "offsets", "emit"]
        seg = []
        for i in range(1, 7):
            a_, b_ = ck[:, i - 1], ck[:, i]
            ok = (a_ > 0) & (b_ > 0)
            if ok.any():
                seg.append(f"{names[i]}={(b_[ok] - a_[ok]).median().item():.0f}")
        if seg:
            print(f"rep{rep} select cycles (t0 warp): " + " ".join(seg))
        lastr = (t[:, 7] > 0) & (ck[:, 8] > 0) & (ck[:, 10] > 0)
        if lastr.any():
            c8, c9, c10, c14 = ck[lastr, 8], ck[lastr, 9], ck[lastr, 10], ck[lastr, 14]
            print(f"rep{rep} combine cycles (last ranks): atomic={(c9 - c8).median().item():.0f} "
                  f"merge={(c10 - c9).median().item():.0f} reset={(c14 - c10).median().item():.0f}")
        nl = (t[:, 7] == 0) & (ck[:, 8] > 0) & (ck[:, 9] > 0)
        if nl.any():
            print(f"rep{rep} atomic cycles (other ranks): {(ck[nl, 9] - ck[nl, 8]).median().item():.0f}")
        for i in (8, 27, 5, 20, 15):
            c = t[:, i]
            if (c > 0).any():
                j = int(torch.argmax(c).item())
                print(f"rep{rep} slowest at {NAMES.get(i, i)}: cta {j} (rank {j % M}, unit {j // M}) "
                      f"+{(c[j] - c[c > 0].median()).item() / 1e3:.2f} us over median")
        print(f"rep{rep} " + " ".join(f"{nm}={md:.2f}/{mx:.2f}" for md, mx, nm in cols))
    H._lib.check(H.lib().hata_debug_trace(None), "trace off")


if __name__ == "__main__":
    main()
