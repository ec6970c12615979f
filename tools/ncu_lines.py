"""Attribute ncu warp-stall samples (SASS source page) to CUDA source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep OBJ_OR_CUBIN KERNEL_MANGLED_SUBSTR [top]
env:   SORT=inst  sort by executed instructions instead of stall samples
       PHASES=1   also sum samples per kernel phase (HATA_TRACE markers in
                  hata_decode_kernel.cuh delimit the phases)

Runs `ncu -i --page source --csv` (SASS view), `cuobjdump -xelf` + `nvdisasm -g`
for line info, maps instruction offsets (runtime address - function start) to
(file, line), and prints the top lines with their two largest stall reasons.
Dev tooling only.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "..", "paper_2506_02572_b200", "csrc")


def main():
    rep, obj, kern = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    hdr = rows[hi]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_x = hdr.index("Instructions Executed")
    reasons = [(j, h) for j, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    i_wx = hdr.index("L1 Wavefronts Shared Excessive") if "L1 Wavefronts Shared Excessive" in hdr else None
    data = [r for r in rows[hi + 1:] if len(r) > i_s and r[0].startswith("0x")]
    base = min(int(r[0], 16) for r in data)
    tmp = tempfile.mkdtemp()
    if obj.endswith(".cubin"):
        cub = obj
    else:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
        cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
    sass = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    lines = sass.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kern in l)
    off2line = {}
    cur = ("?", 0)
    for l in lines[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m:
            off2line[int(m.group(1), 16)] = cur
    agg = collections.Counter()
    ex = collections.Counter()
    wx = collections.Counter()
    why = collections.defaultdict(collections.Counter)
    tot = 0.0
    for r in data:
        key = off2line.get(int(r[0], 16) - base, ("?", 0))
        s = float(r[i_s] or 0)
        agg[key] += s
        ex[key] += float(r[i_x] or 0)
        if i_wx is not None:
            wx[key] += float(r[i_wx] or 0)
        for j, h in reasons:
            why[key][h[6:]] += float(r[j] or 0)
        tot += s
    srcfiles = {}

    def text_of(f, ln):
        for cand in glob.glob(os.path.join(CSRC, f)):
            srcfiles.setdefault(cand, open(cand).read().splitlines())
            if 0 < ln <= len(srcfiles[cand]):
                return srcfiles[cand][ln - 1].strip()
        return ""

    if os.environ.get("PHASES"):
        kf = os.path.join(CSRC, "hata_decode_kernel.cuh")
        marks = []
        for i, l in enumerate(open(kf).read().splitlines(), 1):
            m = re.search(r"HATA_TRACE\((\d+)\)", l)
            if m:
                marks.append((i, int(m.group(1))))
        ph = collections.Counter()
        for (f, ln), s in agg.items():
            if f != "hata_decode_kernel.cuh":
                ph[f] += s
                continue
            name = "pre"
            for mln, mid in marks:
                if ln >= mln:
                    name = f"after_trace{mid}"
            ph[name] += s
        print("per phase (stall samples %):")
        for k, v in sorted(ph.items(), key=lambda kv: -kv[1]):
            print(f"  {v / tot * 100:5.1f}%  {k}")
    order = agg.most_common(top) if os.environ.get("SORT") != "inst" else [(k2, agg[k2]) for k2, _ in ex.most_common(top)]
    for (f, ln), s in order:
        rs = ", ".join(f"{k}={v / max(s, 1) * 100:.0f}%" for k, v in why[(f, ln)].most_common(2))
        extra = f" smem_excess={wx[(f, ln)]:.0f}" if wx[(f, ln)] else ""
        print(f"{s / tot * 100:5.1f}%  inst={ex[(f, ln)]:8.0f}  {f}:{ln:<4d} [{rs}]{extra}  {text_of(f, ln)[:80]}")


if __name__ == "__main__":
    main()
