"""Per-phase timeline of the fused decode kernel (dev tool, needs a GPU).

python tools/trace_decode.py [cfg4] [reps]
Prints, per phase boundary, the median / max over CTAs of (stamp - kernel start)
in microseconds, using hata_debug_trace() (%globaltimer stamps).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402

NAMES = ["start", "qhash", "score", "hist_x", "D_staged", "select", "attn", "end"]


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    sh = synth.CONFIGS[cfg]
    dev = torch.device("cuda", 0)
    sets = [bench.Step(sh, 2000 + i, dev) for i in range(8)]
    H = sets[0].H
    M = H.decode_ranks(sh.B, sh.Hq, sh.Hkv, sh.d, sh.rbits, sh.N, sh.k, sets[0].K.dtype)
    nct = M * sh.B * sh.Hkv
    buf = torch.zeros(nct * 16, dtype=torch.int64, device=dev)
    for s in sets:
        s.run()
    torch.cuda.synchronize()
    H._lib.check(H.lib().hata_debug_trace(buf.data_ptr()), "trace")
    rows = []
    for rep in range(reps):
        s = sets[rep % len(sets)]
        buf.zero_()
        s.decode()
        torch.cuda.synchronize()
        t = buf.view(nct, 16)[:, :8].cpu().double()
        t0 = t[:, 0].min()
        rows.append((t - t0) / 1e3)
    H._lib.check(H.lib().hata_debug_trace(None), "trace off")
    print(f"{cfg}: M={M} ranks x {sh.B * sh.Hkv} units = {nct} CTAs")
    for rep, t in enumerate(rows):
        valid = t[:, 7] > 0
        parts = []
        for i, nm in enumerate(NAMES):
            col = t[:, i][t[:, i] >= 0]
            parts.append(f"{nm}={col.median().item():6.2f}/{col.max().item():6.2f}")
        print(f"rep{rep} " + " ".join(parts))


if __name__ == "__main__":
    main()
